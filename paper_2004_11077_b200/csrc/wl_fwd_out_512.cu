// Output-side forward passes for 512 padded output channels (wl_fwd_out.inc).
#define WL_LD 512
#include "wl_fwd_out.inc"
