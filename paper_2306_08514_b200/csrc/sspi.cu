// Sparse interpolation map (SSPI-SRP) on sm_100a:
//   z[f][i] = sum_p sum_{w < W_p} v[p][i][w] * xi[s[p][i][w]][f]
// restating interpolation.py:188-195 (_dot_sparse_rows :121-126).  With a
// keep-all operator the same kernel is si_map (:129-136), so sspi(all) == si
// bit-for-bit as in the reference (interpolation.py:112-126).
//
// Operator (built once on the host from the reference CSR): pair-major ELL with
// rows padded to a multiple of 32 candidates.  Entries of pair p live at
// ell[ell_off[p] + i * W_p + w] as packed (float value bits, absolute sample index);
// padding entries carry value 0.  Each (candidate, pair) keeps the reference's
// entries in ascending column order.
//
// Samples are lag-major: xi[s][f] with row pitch `ld` (frames contiguous), as
// written by the fused frontend.  Tile kernel: a CTA owns 32 candidates x 128
// frames.  The CTA's operator rows (one contiguous run per pair) are staged in
// shared memory by TMA bulk copies (cp.async.bulk + mbarrier); each lane owns
// 4 consecutive frames and each warp 4 candidates, so every kept entry is one
// broadcast shared-memory read of (value, lag), one coalesced 16-byte read of
// xi[lag][f..f+3] (L1-resident across the CTA) and 4 FMAs into registers.  The
// pair sum stays in registers; z is written through a shared-memory transpose as
// coalesced rows z[f][i0 : i0+32] and the per-frame argmax is folded into packed
// 64-bit keys (one atomicMax per frame per CTA).
#include "common.cuh"

namespace srpgpu {

constexpr int kSspiWarps = 8;
constexpr int kSspiG = 4;                          // candidates per warp
constexpr int kSspiTI = kSspiWarps * kSspiG;       // 32 candidates per CTA
constexpr int kSspiTF = 128;                       // frames per CTA (4 per lane)
constexpr int kSspiOpsBudget = 96 * 1024;          // bytes of staged operator rows per chunk

struct SspiParams {
  const float* xi;           // [S][ld]
  int64_t ld;
  int64_t F;
  int32_t S;
  int32_t P;
  const int32_t* widths;     // [P]
  const int64_t* ell_off;    // [P+1]
  const uint2* ell;          // packed entries, rows padded to a multiple of 32
  int64_t J;
  float* z;                  // [F][J] or null
  unsigned long long* keys;  // [F] or null
  int32_t ent_max;           // max sum of widths per staged chunk
};

__device__ __forceinline__ uint32_t s_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kSspiWarps * 32)
sspi_tile_kernel(const SspiParams prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  int* s_w = reinterpret_cast<int*>(smem_raw);                                  // [P]
  float* zs = reinterpret_cast<float*>(smem_raw + (((size_t)prm.P * 4 + 127) & ~(size_t)127));  // [TF][TI+1]
  uint2* ops = reinterpret_cast<uint2*>(
      reinterpret_cast<unsigned char*>(zs) + (((size_t)kSspiTF * (kSspiTI + 1) * 4 + 127) & ~(size_t)127));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * kSspiTI;
  const int64_t f0 = (int64_t)blockIdx.y * kSspiTF;
  const int P = prm.P;
  for (int i = tid; i < P; i += blockDim.x) s_w[i] = prm.widths[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  float acc[kSspiG][4];
#pragma unroll
  for (int c = 0; c < kSspiG; ++c)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[c][t] = 0.f;
  const int64_t fl = f0 + 4 * lane;
  const bool lane_ok = fl < prm.ld;
  const float* xcol = prm.xi + fl;

  uint32_t phase = 0;
  int pc0 = 0;
  while (pc0 < P) {
    int pc1 = pc0, ents = 0;
    while (pc1 < P && (pc1 == pc0 || ents + s_w[pc1] <= prm.ent_max)) ents += s_w[pc1++];
    if (ents > 0) {
      if (tid == 0) {
        // TMA bulk copies: this CTA's rows of every pair in the chunk
        const uint32_t bytes = (uint32_t)ents * kSspiTI * 8u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(&bar)), "r"(bytes)
                     : "memory");
        int e = 0;
        for (int p = pc0; p < pc1; ++p) {
          const int W = s_w[p];
          if (W == 0) continue;
          const uint2* src = prm.ell + prm.ell_off[p] + i0 * W;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  s_addr(ops + (size_t)e * kSspiTI)),
              "l"(src), "r"((uint32_t)(W * kSspiTI * 8)), "r"(s_addr(&bar))
              : "memory");
          e += W;
        }
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n\t}" ::"r"(s_addr(&bar)),
          "r"(phase)
          : "memory");
      phase ^= 1u;
      if (lane_ok) {
        const uint2* opp = ops;
        for (int p = pc0; p < pc1; ++p) {
          const int W = s_w[p];
          const uint2* rowb = opp + (warp * kSspiG) * W;
#pragma unroll 2
          for (int w = 0; w < W; ++w) {
            uint2 en[kSspiG];
            float4 x[kSspiG];
#pragma unroll
            for (int c = 0; c < kSspiG; ++c) en[c] = rowb[c * W + w];
#pragma unroll
            for (int c = 0; c < kSspiG; ++c)
              x[c] = __ldg(reinterpret_cast<const float4*>(xcol + (int64_t)en[c].y * prm.ld));
#pragma unroll
            for (int c = 0; c < kSspiG; ++c) {
              const float v = __uint_as_float(en[c].x);
              acc[c][0] = fmaf(v, x[c].x, acc[c][0]);
              acc[c][1] = fmaf(v, x[c].y, acc[c][1]);
              acc[c][2] = fmaf(v, x[c].z, acc[c][2]);
              acc[c][3] = fmaf(v, x[c].w, acc[c][3]);
            }
          }
          opp += (size_t)W * kSspiTI;
        }
      }
      __syncthreads();   // the next chunk overwrites `ops`
    }
    pc0 = pc1;
  }

  // epilogue: transpose through shared memory -> coalesced rows of z, fused argmax
#pragma unroll
  for (int c = 0; c < kSspiG; ++c)
#pragma unroll
    for (int t = 0; t < 4; ++t) zs[(4 * lane + t) * (kSspiTI + 1) + warp * kSspiG + c] = acc[c][t];
  __syncthreads();
  const int ti_valid = (int)(prm.J - i0 < kSspiTI ? prm.J - i0 : kSspiTI);
  for (int row = warp; row < kSspiTF; row += kSspiWarps) {
    const int64_t fg = f0 + row;
    if (fg >= prm.F) break;
    unsigned long long key = 0ull;
    if (lane < ti_valid) {
      const float v = zs[row * (kSspiTI + 1) + lane];
      if (prm.z) prm.z[fg * prm.J + i0 + lane] = v;
      key = make_key(v, (uint32_t)(i0 + lane));
    }
    if (prm.keys) {
      key = warp_key_max(key);
      if (lane == 0) atomicMax(prm.keys + fg, key);
    }
  }
}

// Small-frame-count path (e.g. the per-frame reference call): a thread per
// (candidate, frame), entries read straight from global memory.
__global__ void sspi_rows_kernel(const SspiParams prm) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t f = blockIdx.y;
  const bool live = gi < prm.J;
  float acc = 0.f;
  if (live) {
    for (int p = 0; p < prm.P; ++p) {
      const int W = prm.widths[p];
      const uint2* e = prm.ell + prm.ell_off[p] + gi * W;
      for (int w = 0; w < W; ++w) {
        const uint2 en = e[w];
        acc = fmaf(__uint_as_float(en.x), __ldg(prm.xi + (int64_t)en.y * prm.ld + f), acc);
      }
    }
    if (prm.z) prm.z[f * prm.J + gi] = acc;
  }
  if (prm.keys) {
    unsigned long long key = live ? make_key(acc, (uint32_t)gi) : 0ull;
    key = warp_key_max(key);
    if ((threadIdx.x & 31) == 0 && key) atomicMax(prm.keys + f, key);
  }
}

// out[c][r] = in[r][c]: frame-major samples [F][S] -> lag-major [S][ld]
__global__ void transpose_kernel(const float* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                 float* __restrict__ out, int64_t ld_out) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    t[j][threadIdx.x] = (r < rows && c < cols) ? in[r * ld_in + c] : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (c < cols && r < ld_out) out[c * ld_out + r] = (r < rows) ? t[threadIdx.x][j] : 0.f;
  }
}

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_sspi_map(const float* samples, int64_t samples_ld, int64_t num_frames,
                               int32_t total_samples, int32_t num_pairs, const int32_t* widths,
                               const int64_t* ell_offsets, const void* ell, int64_t num_candidates,
                               int32_t max_width, int32_t sum_widths, float* z, uint64_t* keys,
                               srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_pairs >= 1 && num_candidates >= 1 && total_samples >= 1, SRPGPU_ERR_DIMENSION,
                   "sspi_map: empty operator");
  SRPGPU_CHECK_ARG(num_candidates < 0xFFFFFFFFll, SRPGPU_ERR_DIMENSION, "sspi_map: too many candidates");
  SRPGPU_CHECK_ARG(samples_ld >= num_frames && samples_ld % 4 == 0, SRPGPU_ERR_VALUE,
                   "sspi_map: lag-major pitch must cover the frames and be a multiple of 4");
  SRPGPU_CHECK_ARG(((uintptr_t)samples & 15) == 0 && ((uintptr_t)ell & 15) == 0, SRPGPU_ERR_VALUE,
                   "sspi_map: operands must be 16-byte aligned");
  if (num_frames <= 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  SspiParams prm = {};
  prm.xi = samples; prm.ld = samples_ld; prm.F = num_frames; prm.S = total_samples; prm.P = num_pairs;
  prm.widths = widths; prm.ell_off = ell_offsets;
  prm.ell = reinterpret_cast<const uint2*>(ell); prm.J = num_candidates; prm.z = z;
  prm.keys = reinterpret_cast<unsigned long long*>(keys);
  if (keys) {
    if (cudaMemsetAsync(keys, 0, (size_t)num_frames * sizeof(uint64_t), st) != cudaSuccess) {
      set_error("sspi_map: key reset failed");
      return SRPGPU_ERR_LAUNCH;
    }
  }
  if (num_frames < 32) {
    dim3 grid((unsigned)((num_candidates + 255) / 256), (unsigned)num_frames);
    sspi_rows_kernel<<<grid, 256, 0, st>>>(prm);
    SRPGPU_CHECK_LAUNCH("sspi_map(rows)");
    return SRPGPU_OK;
  }
  const int ent_cap = kSspiOpsBudget / (kSspiTI * 8);
  prm.ent_max = std::max(std::max(max_width, 1), std::min(std::max(sum_widths, 1), ent_cap));
  const size_t smem = (((size_t)num_pairs * 4 + 127) & ~(size_t)127) +
                      (((size_t)kSspiTF * (kSspiTI + 1) * 4 + 127) & ~(size_t)127) +
                      (size_t)prm.ent_max * kSspiTI * 8;
  SRPGPU_CHECK_ARG(smem <= 227 * 1024, SRPGPU_ERR_UNSUPPORTED,
                   "sspi_map: ELL width %d needs %zu B shared memory", max_width, smem);
  if (cudaFuncSetAttribute(sspi_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("sspi_map: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  SRPGPU_CHECK_ARG((num_frames + kSspiTF - 1) / kSspiTF <= 65535, SRPGPU_ERR_DIMENSION,
                   "sspi_map: too many frames per call");
  dim3 grid((unsigned)((num_candidates + kSspiTI - 1) / kSspiTI),
            (unsigned)((num_frames + kSspiTF - 1) / kSspiTF));
  sspi_tile_kernel<<<grid, kSspiWarps * 32, smem, st>>>(prm);
  SRPGPU_CHECK_LAUNCH("sspi_map");
  return SRPGPU_OK;
}

extern "C" int srpgpu_transpose(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                                int64_t ld_dst, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(ld_src >= cols && ld_dst >= rows, SRPGPU_ERR_DIMENSION, "transpose: bad pitches");
  if (rows <= 0 || cols <= 0) return SRPGPU_OK;
  SRPGPU_CHECK_ARG((ld_dst + 31) / 32 <= 65535, SRPGPU_ERR_DIMENSION, "transpose: too many rows");
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((ld_dst + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, rows, cols, ld_src, dst, ld_dst);
  SRPGPU_CHECK_LAUNCH("transpose");
  return SRPGPU_OK;
}
