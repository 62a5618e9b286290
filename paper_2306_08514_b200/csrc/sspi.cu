// Sparse interpolation map (SSPI-SRP) on sm_100a:
//   z[f][i] = sum_p sum_{w < W_p} v[p][i][w] * xi[f][s[p][i][w]]
// restating interpolation.py:188-195 (_dot_sparse_rows :121-126).  With a
// keep-all operator the same kernel is si_map (:129-136), so sspi(all) == si
// bit-for-bit as in the reference (interpolation.py:112-126).
//
// Operator layout (built once on the host from the reference CSR): pair-major
// ELL.  Entries of pair p live at ell[ell_off[p] + i * W_p + w] as packed
// (float value bits, absolute sample index s = offsets[p] + column-in-pair);
// padding entries carry value 0 and a valid index.  Each (candidate, pair)
// keeps the reference's entries in ascending column order.
//
// Frame-tiled kernel: lanes own frames (4 consecutive frames per lane, one
// 16-byte shared-memory read per kept entry), warps own G candidates each.
// The CTA stages a chunk of pair blocks of xi (lags x 128 frames) and the
// operator slice of its candidates in shared memory, accumulates the pair sum
// in registers across all pairs, then writes z through a shared-memory transpose
// (coalesced rows of z[f][i0 : i0+TI]) and folds the per-frame argmax into a
// packed 64-bit key with one atomicMax per frame per CTA.
#include "common.cuh"

namespace srpgpu {

constexpr int kSspiThreads = 256;  // 8 warps
constexpr int kSspiFpt = 4;        // frames per lane
constexpr int kSspiTF = 32 * kSspiFpt;  // frames per CTA tile = 128
constexpr int kSspiRowStride = kSspiTF + 4;  // padded smem row (floats)

struct SspiParams {
  const float* xi;           // [F][S]
  int64_t F;
  int32_t S;
  int32_t P;
  const int32_t* offsets;    // [P+1]
  const int32_t* widths;     // [P]
  const int64_t* ell_off;    // [P+1]
  const uint2* ell;          // packed entries
  int64_t J;
  float* z;                  // [F][J] or null
  unsigned long long* keys;  // [F] or null
  int32_t rows_max;          // xi rows per smem chunk
  int32_t ent_max;           // operator entries per (candidate) per chunk, upper bound
};

template <int G>
__global__ void __launch_bounds__(kSspiThreads)
sspi_tile_kernel(const SspiParams prm) {
  constexpr int TI = 8 * G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* s_off = reinterpret_cast<int*>(smem_raw);            // [P+1]
  int* s_w = s_off + (prm.P + 1);                            // [P]
  long long* s_eoff = reinterpret_cast<long long*>(
      smem_raw + (((size_t)(2 * prm.P + 1) * sizeof(int) + 15) & ~(size_t)15));  // [P+1]
  float* xs = reinterpret_cast<float*>(
      reinterpret_cast<unsigned char*>(s_eoff) + (((size_t)(prm.P + 1) * 8 + 15) & ~(size_t)15));
  uint2* ops = reinterpret_cast<uint2*>(xs + (size_t)prm.rows_max * kSspiRowStride);  // [TI][ent_max]
  float* zs = reinterpret_cast<float*>(ops + (size_t)TI * prm.ent_max);              // [TF][TI+1]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t f0 = (int64_t)blockIdx.y * kSspiTF;
  const int P = prm.P;

  for (int i = tid; i <= P; i += blockDim.x) {
    s_off[i] = prm.offsets[i];
    s_eoff[i] = prm.ell_off[i];
  }
  for (int i = tid; i < P; i += blockDim.x) s_w[i] = prm.widths[i];
  __syncthreads();

  float acc[G][kSspiFpt];
#pragma unroll
  for (int c = 0; c < G; ++c)
#pragma unroll
    for (int t = 0; t < kSspiFpt; ++t) acc[c][t] = 0.f;

  int pc0 = 0;
  while (pc0 < P) {
    // chunk of pairs whose lag blocks fit the staging buffer (uniform across the CTA)
    int pc1 = pc0 + 1;
    int ents = s_w[pc0];
    while (pc1 < P && s_off[pc1 + 1] - s_off[pc0] <= prm.rows_max && ents + s_w[pc1] <= prm.ent_max) {
      ents += s_w[pc1];
      ++pc1;
    }
    const int base = s_off[pc0];
    const int rows = s_off[pc1] - base;
    // stage xi[f0 : f0+TF][base : base+rows] transposed to xs[row][frame]
    for (int idx = tid; idx < rows * kSspiTF; idx += blockDim.x) {
      const int f = idx / rows, r = idx - f * rows;
      const int64_t fg = f0 + f;
      xs[r * kSspiRowStride + f] = (fg < prm.F) ? __ldg(prm.xi + fg * prm.S + base + r) : 0.f;
    }
    // stage the operator slice: candidate-major, pairs of the chunk back to back
    for (int idx = tid; idx < TI * ents; idx += blockDim.x) {
      const int c = idx / ents;
      int e = idx - c * ents;
      int p = pc0;
      while (e >= s_w[p]) { e -= s_w[p]; ++p; }
      const int64_t i = i0 + c;
      uint2 v = make_uint2(0u, (unsigned)base);
      if (i < prm.J) v = prm.ell[s_eoff[p] + i * s_w[p] + e];
      ops[c * prm.ent_max + (idx - c * ents)] = v;
    }
    __syncthreads();
    const float* xl = xs + lane * kSspiFpt;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const uint2* oc = ops + (warp * G + c) * prm.ent_max;
      for (int e = 0; e < ents; ++e) {
        const uint2 en = oc[e];
        const float v = __uint_as_float(en.x);
        const float4 x = *reinterpret_cast<const float4*>(xl + ((int)en.y - base) * kSspiRowStride);
        acc[c][0] = fmaf(v, x.x, acc[c][0]);
        acc[c][1] = fmaf(v, x.y, acc[c][1]);
        acc[c][2] = fmaf(v, x.z, acc[c][2]);
        acc[c][3] = fmaf(v, x.w, acc[c][3]);
      }
    }
    __syncthreads();
    pc0 = pc1;
  }

  // epilogue: transpose through shared memory -> coalesced rows of z, fused argmax
#pragma unroll
  for (int c = 0; c < G; ++c)
#pragma unroll
    for (int t = 0; t < kSspiFpt; ++t) zs[(lane * kSspiFpt + t) * (TI + 1) + warp * G + c] = acc[c][t];
  __syncthreads();
  const int ti_valid = (int)(prm.J - i0 < TI ? prm.J - i0 : TI);
  for (int row = warp; row < kSspiTF; row += kSspiThreads / 32) {
    const int64_t fg = f0 + row;
    if (fg >= prm.F) break;
    unsigned long long key = 0ull;
    for (int c = lane; c < ti_valid; c += 32) {
      const float v = zs[row * (TI + 1) + c];
      if (prm.z) prm.z[fg * prm.J + i0 + c] = v;
      key = key_max(key, make_key(v, (uint32_t)(i0 + c)));
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
    const float* x = prm.xi + f * prm.S;
    for (int p = 0; p < prm.P; ++p) {
      const int W = prm.widths[p];
      const uint2* e = prm.ell + prm.ell_off[p] + gi * W;
      for (int w = 0; w < W; ++w) {
        const uint2 en = e[w];
        acc = fmaf(__uint_as_float(en.x), __ldg(x + en.y), acc);
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

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_sspi_map(const float* samples, int64_t num_frames, int32_t total_samples,
                               int32_t num_pairs, const int32_t* offsets, const int32_t* widths,
                               const int64_t* ell_offsets, const void* ell, int64_t num_candidates,
                               int32_t max_block, int32_t max_width, int32_t sum_widths, float* z,
                               uint64_t* keys,
                               srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_pairs >= 1 && num_candidates >= 1 && total_samples >= 1, SRPGPU_ERR_DIMENSION,
                   "sspi_map: empty operator");
  SRPGPU_CHECK_ARG(num_candidates < 0xFFFFFFFFll, SRPGPU_ERR_DIMENSION, "sspi_map: too many candidates");
  if (num_frames <= 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  SspiParams prm = {};
  prm.xi = samples; prm.F = num_frames; prm.S = total_samples; prm.P = num_pairs;
  prm.offsets = offsets; prm.widths = widths; prm.ell_off = ell_offsets;
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
  constexpr int G = 4, TI = 8 * G;
  const int rows_max = std::max(max_block, std::min(total_samples, 96));
  // a chunk always holds at least one whole pair block
  prm.rows_max = rows_max;
  prm.ent_max = std::max(std::max(max_width, 1), std::min(sum_widths, 128));
  size_t head = (((size_t)(2 * num_pairs + 1) * sizeof(int) + 15) & ~(size_t)15) +
                (((size_t)(num_pairs + 1) * 8 + 15) & ~(size_t)15);
  size_t smem = head + (size_t)rows_max * kSspiRowStride * sizeof(float) +
                (size_t)TI * prm.ent_max * sizeof(uint2) + (size_t)kSspiTF * (TI + 1) * sizeof(float);
  SRPGPU_CHECK_ARG(smem <= 227 * 1024, SRPGPU_ERR_UNSUPPORTED,
                   "sspi_map: pair block of %d lags needs %zu B shared memory", max_block, smem);
  auto kern = sspi_tile_kernel<G>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("sspi_map: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  dim3 grid((unsigned)((num_candidates + TI - 1) / TI), (unsigned)((num_frames + kSspiTF - 1) / kSspiTF));
  kern<<<grid, kSspiThreads, smem, st>>>(prm);
  SRPGPU_CHECK_LAUNCH("sspi_map");
  return SRPGPU_OK;
}
