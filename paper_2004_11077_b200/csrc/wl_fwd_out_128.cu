// Output-side forward passes for 128 padded output channels (wl_fwd_out.inc).
#define WL_LD 128
#include "wl_fwd_out.inc"
