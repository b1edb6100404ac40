// The phase-A tensor-core GEMM built with 128-row tiles and four TMEM
// accumulators (see vs_tc.cu): used for the IVF coarse quantizer.
#define VS_TC_BN 128
#define VS_TC_NS bn128
#define VS_TC_INLINE
#include "vs_tc.cu"
