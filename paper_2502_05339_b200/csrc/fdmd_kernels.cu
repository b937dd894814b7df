// B200 (sm_100a) kernels for the DMD hot path (see fdmd_kernels.cuh):
//   fdmd_tall.cuh    FP64 DMMA contractions (tall_gemm, tall_gram)
//   fdmd_stream.cuh  HBM-streaming reconstruction and helper kernels
//   fdmd_mac.cuh     2-D MAC-grid serving / upscaling kernels
#include "fdmd_kernels.cuh"

#include <cfloat>
#include <climits>
#include <cstdio>

#include "fdmd_tall.cuh"
#include "fdmd_tall_tma.cuh"
#include "fdmd_gram_tma.cuh"
#include "fdmd_gram_panel.cuh"
#include "fdmd_tc_decode.cuh"
#include "fdmd_tc_decode2.cuh"
#include "fdmd_stream.cuh"
#include "fdmd_mac.cuh"
#include "fdmd_solver.cuh"
