// Input-side forward passes for 512 padded channels (wl_fwd_in.inc).
#define WL_LD 512
#include "wl_fwd_in.inc"
