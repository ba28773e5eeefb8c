// Output-side forward passes for 64 padded output channels (wl_fwd_out.inc).
#define WL_LD 64
#include "wl_fwd_out.inc"
