// Output-side forward passes for 256 padded output channels (wl_fwd_out.inc).
#define WL_LD 256
#include "wl_fwd_out.inc"
