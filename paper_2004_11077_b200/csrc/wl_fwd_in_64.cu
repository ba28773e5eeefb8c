// Input-side forward passes for 64 padded channels (wl_fwd_in.inc).
#define WL_LD 64
#include "wl_fwd_in.inc"
