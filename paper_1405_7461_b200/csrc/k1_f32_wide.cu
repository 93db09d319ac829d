// k1_f32_wide.cu — the FP32 K1 kernel (k1_f32.cu) built for the largest
// plans: 1,024-query tiles holding octets of Periodic batches (a staircase of
// up to 15 candidate segments per group of 8), 16-warp CTAs at up to 128
// registers, one CTA per SM (the tile's shared memory does not fit twice;
// the window arrays are padded to K1_TQ + 64 so that 16 warps fit).
// A candidate sub-tile visit then serves up to 8 batches instead of 4: about
// half the per-visit cost (group data, window, box cull, staging) per pair.
// search.cu picks it for plans of >= kWideMinBatches batches.
#define K1_WIDE 1
#define K1_TQ_DEF 1024
#ifndef K1W_THREADS_DEF
#define K1W_THREADS_DEF 512
#endif
#define K1_THREADS_DEF K1W_THREADS_DEF
#define K1F_MIN_BLOCKS 1
#define K1_GMAX_DEF 8
#include "k1_f32.cu"
