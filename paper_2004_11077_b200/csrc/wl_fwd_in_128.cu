// Input-side forward passes for 128 padded channels (wl_fwd_in.inc).
#define WL_LD 128
#include "wl_fwd_in.inc"
