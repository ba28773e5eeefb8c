// Input-side forward passes for 32 padded channels (wl_fwd_in.inc).
#define WL_LD 32
#include "wl_fwd_in.inc"
