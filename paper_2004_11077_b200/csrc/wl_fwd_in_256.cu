// Input-side forward passes for 256 padded channels (wl_fwd_in.inc).
#define WL_LD 256
#include "wl_fwd_in.inc"
