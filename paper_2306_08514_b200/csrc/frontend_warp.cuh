// Parameters of the warp-per-frame frontend (frontend_warp.cu), shared with frontend.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

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
  int32_t planes_tf32;  // 1: planes are fp32 hi = tf32_rne(x), lo = tf32_rne(x - hi); 2: fp16 hi = f16_rne(x),
                        // lo = f16_rne(x - hi) (both lag-major only; fp16 needs |x| in fp16 range: PHAT)
};

// PHAT weighting raw / max(|raw|, floor), 0 where that is 0 (frontend.py:154-158), with the
// per-frame constants hoisted: rsqrt(|raw|^2) above the floor, 1 / floor below it.
struct Phat {
  int weighting;
  float floor2, inv_floor;
  __device__ __forceinline__ Phat(int w, float floor)
      : weighting(w), floor2(floor * floor), inv_floor(floor > 0.f ? 1.0f / floor : 0.f) {}
  __device__ __forceinline__ float2 operator()(float2 raw) const {
    if (weighting) {
      const float mag2 = raw.x * raw.x + raw.y * raw.y;
      const float inv = (mag2 > floor2 && mag2 > 0.f) ? rsqrtf(mag2) : inv_floor;
      raw.x *= inv;
      raw.y *= inv;
    }
    return raw;
  }
};

// one xi sample (storage index d of a pair block at offset o with N lags a side): the
// f32 output and, when requested, its bf16 hi/lo planes (storage or natural lag order)
__device__ __forceinline__ void put_xi(const WarpParams& prm, float* dst, int64_t sst, int64_t f, int o, int N, int d,
                                       float v) {
  dst[(o + d) * sst] = v;
  if (prm.xi_planes) {
    const int col = o + (prm.xi_natural ? (d <= N ? N + d : d - N - 1) : d);
    if (prm.planes_tf32 == 2) {               // lag-major fp16 [2][cols8][planes_ld]
      __half* pl = reinterpret_cast<__half*>(prm.xi_planes) + (int64_t)col * prm.planes_ld + f;
      const __half hi = __float2half_rn(v);
      pl[0] = hi;
      pl[(int64_t)prm.cols8 * prm.planes_ld] = __float2half_rn(v - __half2float(hi));
      return;
    }
    if (prm.planes_tf32) {                    // lag-major fp32 [2][cols8][planes_ld]
      float* pl = reinterpret_cast<float*>(prm.xi_planes) + (int64_t)col * prm.planes_ld + f;
      const float hi = tf32_rne(v);
      pl[0] = hi;
      pl[(int64_t)prm.cols8 * prm.planes_ld] = tf32_rne(v - hi);
      return;
    }
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(prm.xi_planes);
    if (prm.planes_ld) {                      // lag-major [2][cols8][planes_ld]
      __nv_bfloat16* pl = base + (int64_t)col * prm.planes_ld + f;
      pl[0] = hi;
      pl[(int64_t)prm.cols8 * prm.planes_ld] = lo;
    } else {
      __nv_bfloat16* pl = base + f * prm.cols8 + col;
      pl[0] = hi;
      pl[prm.F * prm.cols8] = lo;
    }
  }
}

// Sliced-ELL sparse interpolation operator + outputs of the fused frames -> SSPI map chain.
struct SellMap {
  const uint16_t* cols;      // [sum_c W_c][32] sample index per entry (chunk c = candidates 32c..32c+31)
  const float* vals;         // [sum_c W_c][32] weight (0 in padding entries)
  const int32_t* chunk_off;  // [ceil(J/32) + 1] first entry row of each chunk
  int64_t J;
  float* z;                  // [F][J] or null
  int64_t* index;            // [F] argmax index or null
  uint64_t* keys;            // [F] packed argmax keys or null
};

// SLRI factors + outputs of the fused frames -> SLRI map chain.
struct SlriMap {
  const float* fat;          // [R][S]
  const float* tallT;        // [round16(R)][J] (tall transposed: candidates contiguous; rows >= R zero)
  int32_t R, S;
  int64_t J;
  float* z;                  // [F][J] or null
  int64_t* index;            // [F] argmax index or null
  uint64_t* keys;            // [F] packed argmax keys or null
};

// frontend + SSPI / SLRI map + argmax in one launch (frame lengths 256 / 512 / 1024).
int frontend_sspi_launch(const WarpParams& wp, const SellMap& mp, cudaStream_t st, const char* what);
int frontend_slri_launch(const WarpParams& wp, const SlriMap& mp, cudaStream_t st, const char* what);

// 0: launched; 1: shape not covered (use the block kernel); < 0: error status.
int frontend_warp_launch(const WarpParams& wp, int out, cudaStream_t st, const char* what);

// Task-per-warp frontend (frontend_lane.cu): same contract as frontend_warp_launch.
int frontend_lane_launch(const WarpParams& wp, int out, cudaStream_t st, const char* what);

// Frontend kernel choice: 0 auto (by batch size), 1 warp-per-frame, 2 task-per-warp, 3 block.
int frontend_kernel_choice();

}  // namespace srpgpu
