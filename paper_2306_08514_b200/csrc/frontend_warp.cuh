// Parameters of the warp-per-frame frontend (frontend_warp.cu), shared with frontend.cu.
#pragma once
#include "common.cuh"

namespace srpgpu {

enum { W_OUT_GCC = 1, W_OUT_XI = 2 };

struct WarpParams {
  const float* samples;
  int64_t ld_samples;
  const float* window;
  int32_t M, L, K, hop;
  int64_t first_frame, F;
  const int32_t* pairs;
  int32_t P;
  int32_t weighting, floor_mode;
  float floor_value;
  const int32_t* counts;
  const int32_t* offsets;
  int32_t S;
  float2* gcc_out;
  int64_t gcc_ld;
  int32_t round_tf32;
  float* xi_out;
  int64_t xi_ld;   // 0: frame-major [F][S]; > 0: lag-major [S][xi_ld]
  // optional bf16 hi/lo planes [2][F][cols8] of xi for the tensor-core interpolation map
  // (interp_tc.cu): hi = bf16_rne(x), lo = bf16_rne(x - hi), zero in [S, cols8)
  uint16_t* xi_planes;
  int32_t cols8;
  int32_t xi_natural;   // planes in natural lag order -N_p..N_p per pair (gathered-window engine)
  int64_t planes_ld;    // 0: planes frame-major [2][F][cols8]; > 0: lag-major [2][cols8][planes_ld]
};

// 0: launched; 1: shape not covered (use the block kernel); < 0: error status.
int frontend_warp_launch(const WarpParams& wp, int out, cudaStream_t st, const char* what);

}  // namespace srpgpu
