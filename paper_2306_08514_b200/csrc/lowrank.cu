// Dense fp32 SIMT products of the SRP-map hot path on sm_100a:
//
//   out[f][i] = alpha * sum_k A[i][k] * B[f][k]     (+ fused per-frame argmax)
//
// One register-tiled kernel (64 x 64 output tile, 4 x 4 per thread, k staged
// through shared memory) serves
//   * slri_map  z = tall (fat xi)            interpolation.py:178-185
//   * lr_map    z = 2 Re(tall (fat psi))     lowrank.py:51-57  (complex folded into
//               real factors of width 2R on the host, once per operator)
//   * the fp32 SIMT conventional map z = 2 Re(H psi)   srp.py:65-71, with H
//               stored as interleaved (Re H, -Im H) rows against psi's (re, im).
// The tcgen05/TMEM tensor-core conventional map lives in conv_tcgen05.cu.
#include "common.cuh"

namespace srpgpu {

constexpr int kGI = 64, kGF = 64, kGK = 16;

// TI x TF output tile (TI * TF = 4096, 256 threads x 4 x 4): 64 x 64, or 32 x 128 for
// factor products with at most 32 rank rows (LR at R = 16: 2R = 32), so no half-empty tiles
template <bool BT, int TI = 64>   // BT: B stored transposed, element (f, k) at B[k * ldb + f]
__global__ void __launch_bounds__(256)
gemm_nt_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
               float* __restrict__ out, int64_t ldo, int64_t I, int64_t F, int64_t K, float alpha,
               unsigned long long* __restrict__ keys, int64_t key_base, int64_t k_chunk) {
  // split-K: CTA z covers k in [z * k_chunk, min(K, (z + 1) * k_chunk)) and writes its
  // partial product to out + z * F * ldo (reduced afterwards in a fixed order)
  const int64_t kbeg = (int64_t)blockIdx.z * k_chunk;
  const int64_t kend = kbeg + k_chunk < K ? kbeg + k_chunk : K;
  out += (int64_t)blockIdx.z * F * ldo;
  constexpr int TF = 4096 / TI, TX = TI / 4;
  __shared__ __align__(16) float As[kGK][TI + 4];
  __shared__ __align__(16) float Bs[kGK][TF + 4];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  // frame tiles run fastest: co-resident CTAs then cover many frames, so their per-frame
  // key atomics spread over many addresses (candidate-fastest order had ~1000 CTAs
  // hammering the same 64 keys); both operands are small and stay L2-resident
  const int64_t f0 = (int64_t)blockIdx.x * TF, i0 = (int64_t)blockIdx.y * TI;
  float acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;

  // the next k-tile is loaded into registers while the current one is multiplied
  // (register double buffering: the global loads' latency hides behind 256 FMAs)
  constexpr int NA = TI * kGK / 256, NB = TF * kGK / 256;
  float ra[NA], rb[NB];
  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const int idx = tid + r * 256;        // over a TI x 16 tile, k fastest
      const int64_t gi = i0 + (idx >> 4), gk = k0 + (idx & 15);
      ra[r] = (gi < I && gk < kend) ? __ldg(A + gi * lda + gk) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const int idx = tid + r * 256;
      if (!BT) {
        const int64_t gf = f0 + (idx >> 4), gk = k0 + (idx & 15);
        rb[r] = (gf < F && gk < kend) ? __ldg(B + gf * ldb + gk) : 0.f;
      } else {                              // frames fastest: coalesced along f
        const int64_t gf = f0 + idx % TF, gkb = k0 + idx / TF;
        rb[r] = (gf < F && gkb < kend) ? __ldg(B + gkb * ldb + gf) : 0.f;
      }
    }
  };
  auto store_tile = [&]() {
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const int idx = tid + r * 256;
      As[idx & 15][idx >> 4] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const int idx = tid + r * 256;
      if (!BT) Bs[idx & 15][idx >> 4] = rb[r];
      else Bs[idx / TF][idx % TF] = rb[r];
    }
  };
  if (kbeg < kend) load_tile(kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += kGK) {
    store_tile();
    __syncthreads();
    if (k0 + kGK < kend) load_tile(k0 + kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][tx * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][ty * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(bv[u], av[v], acc[u][v]);
    }
    __syncthreads();
  }

  // epilogue: rows f = f0 + 4 ty + u, columns i = i0 + 4 tx + v (16-byte streaming stores
  // when the row pitch allows: the maps are written once and never re-read here)
  const bool vec = out && (ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t f = f0 + ty * 4 + u;
    unsigned long long key = 0ull;
    if (f < F) {
      const int64_t ib = i0 + tx * 4;
      if (vec && ib + 3 < I) {
        const float4 v4 = make_float4(alpha * acc[u][0], alpha * acc[u][1], alpha * acc[u][2],
                                      alpha * acc[u][3]);
        __stcs(reinterpret_cast<float4*>(out + f * ldo + ib), v4);
        key = key_max(key_max(make_key(v4.x, (uint32_t)(key_base + ib)),
                              make_key(v4.y, (uint32_t)(key_base + ib + 1))),
                      key_max(make_key(v4.z, (uint32_t)(key_base + ib + 2)),
                              make_key(v4.w, (uint32_t)(key_base + ib + 3))));
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t i = ib + v;
          if (i < I) {
            const float val = alpha * acc[u][v];
            if (out) out[f * ldo + i] = val;
            key = key_max(key, make_key(val, (uint32_t)(key_base + i)));
          }
        }
      }
    }
    if (keys) {
      // reduce over the TX lanes sharing ty
#pragma unroll
      for (int o = TX / 2; o > 0; o >>= 1) key = key_max(key, __shfl_xor_sync(0xffffffffu, key, o));
      if (tx == 0 && f < F && key) atomicMax(keys + f, key);
    }
  }
}

// Rank-space -> candidate product with a small inner dimension (SLRI: K = R,
// interpolation.py:178-185; LR: K = 2R, lowrank.py:51-57):
//     out[f][i] = alpha * sum_k A[i][k] B[f][k],   K <= KB,
// which is output-bound (K FMAs per 4-byte map element), K <= 16 here.  CTA = 64 frames x a run of
// 128-candidate tiles: the frames' B rows stay in shared memory, the next A tile is
// prefetched into registers while the current one is multiplied, z is written with
// coalesced 16-byte streaming stores, and the per-frame argmax is carried in
// registers across the run (one key atomic per frame per CTA).  Thread (tx, ty) owns
// frames 4ty..4ty+3 and candidates 4tx..4tx+3, 64+4tx..64+4tx+3 of each tile.  The k
// order of every sum is 0..K-1, as in gemm_nt.
constexpr int kOF = 64, kOI = 128;

template <int KB>
__global__ void __launch_bounds__(256)
lowrank_out_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                   float* __restrict__ out, int64_t ldo, int64_t I, int64_t F, int K, int tiles_per_cta,
                   float alpha, unsigned long long* __restrict__ keys) {
  __shared__ __align__(16) float Bs[KB][kOF];
  __shared__ __align__(16) float As[2][KB][kOI];
  constexpr int kPer = KB * kOI / 256;            // A elements per thread per tile
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t f0 = (int64_t)blockIdx.x * kOF;
  const int64_t tile0 = (int64_t)blockIdx.y * tiles_per_cta;
  const int64_t ntiles = (I + kOI - 1) / kOI;
  const int nt = (int)(ntiles - tile0 < tiles_per_cta ? ntiles - tile0 : tiles_per_cta);
  for (int e = tid; e < KB * kOF; e += 256) {   // alpha folded into the rank-space operand
    const int f = e / KB, k = e % KB;
    Bs[k][f] = (k < K && f0 + f < F) ? alpha * __ldg(B + (f0 + f) * ldb + k) : 0.f;
  }
  float areg[kPer];
  auto load_a = [&](int t) {
    const int64_t i0 = (tile0 + t) * kOI;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = tid + j * 256, i = e / KB, k = e % KB;
      areg[j] = (k < K && i0 + i < I) ? __ldg(A + (i0 + i) * lda + k) : 0.f;
    }
  };
  auto store_a = [&](int buf) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = tid + j * 256;
      As[buf][e % KB][e / KB] = areg[j];
    }
  };
  // running first maximum per frame over this thread's candidates (ascending index)
  float bval[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  uint32_t bidx[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
  const bool vec = (ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (nt > 0) {
    load_a(0);
    store_a(0);
  }
  __syncthreads();
  for (int t = 0; t < nt; ++t) {
    const int buf = t & 1;
    if (t + 1 < nt) load_a(t + 1);
    float acc[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][ty * 4]);
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][tx * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + tx * 4]);
      const float bv[4] = {b.x, b.y, b.z, b.w};
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(bv[u], av[v], acc[u][v]);
    }
    const int64_t i0 = (tile0 + t) * kOI;
    const uint32_t c0 = (uint32_t)i0 + tx * 4;              // candidates c0..c0+3, c0+64..c0+67
    const bool full = i0 + kOI <= I && vec;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t f = f0 + ty * 4 + u;
      if (f >= F) continue;
      float* row = out + f * ldo;
      if (full) {
        if (out) {
          __stcs(reinterpret_cast<float4*>(row + c0), make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]));
          __stcs(reinterpret_cast<float4*>(row + c0 + 64), make_float4(acc[u][4], acc[u][5], acc[u][6], acc[u][7]));
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint32_t c = c0 + (v & 3) + (v >> 2) * 64;
          if (acc[u][v] > bval[u]) { bval[u] = acc[u][v]; bidx[u] = c; }
        }
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint32_t c = c0 + (v & 3) + (v >> 2) * 64;
          if ((int64_t)c < I) {
            if (out) __stcs(row + c, acc[u][v]);
            if (acc[u][v] > bval[u] || bidx[u] == 0xFFFFFFFFu) { bval[u] = acc[u][v]; bidx[u] = c; }
          }
        }
      }
    }
    if (t + 1 < nt) store_a(buf ^ 1);
    __syncthreads();
  }
  if (keys) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      unsigned long long k = bidx[u] != 0xFFFFFFFFu ? make_key(bval[u], bidx[u]) : 0ull;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) k = key_max(k, __shfl_xor_sync(0xffffffffu, k, o));
      const int64_t f = f0 + ty * 4 + u;
      if (tx == 0 && f < F && k) atomicMax(keys + f, k);
    }
  }
}

// Dispatch for the small-K candidate product; falls back to gemm_nt beyond K = 16.
int gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* out, int64_t ldo,
            int64_t I, int64_t F, int64_t K, float alpha, uint64_t* keys, cudaStream_t st,
            const char* what, bool b_trans, float* split_ws);

static int lowrank_out(const float* A, int64_t lda, const float* B, int64_t ldb, float* out, int64_t ldo,
                       int64_t I, int64_t F, int64_t K, float alpha, uint64_t* keys, cudaStream_t st,
                       const char* what) {
  if (I <= 0 || F <= 0) return SRPGPU_OK;
  // K = 32 (LR at R = 16) needs 119 registers here (2 CTAs/SM) and measured slower than
  // gemm_nt, so only K <= 16 takes this kernel
  if (K > 16) return gemm_nt(A, lda, B, ldb, out, ldo, I, F, K, alpha, keys, st, what, false, nullptr);
  const int64_t ftiles = (F + kOF - 1) / kOF, itiles = (I + kOI - 1) / kOI;
  // enough CTAs for ~4 waves of 148 SMs x 3 resident, each sweeping a run of candidate tiles
  const int64_t want = 12 * (int64_t)num_sms();
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(itiles, (want + ftiles - 1) / ftiles));
  const int64_t per = (itiles + chunks - 1) / chunks;
  chunks = (itiles + per - 1) / per;
  SRPGPU_CHECK_ARG(chunks <= 65535, SRPGPU_ERR_DIMENSION, "%s: too many candidates", what);
  dim3 grid((unsigned)ftiles, (unsigned)chunks);
  auto* kp = reinterpret_cast<unsigned long long*>(keys);
  lowrank_out_kernel<16><<<grid, 256, 0, st>>>(A, lda, B, ldb, out, ldo, I, F, (int)K, (int)per, alpha, kp);
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

// out[f][i] = sum_z part[z][f][i] in a fixed order (deterministic split-K)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int64_t nz, int64_t n,
                                     float* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t z = 0; z < nz; ++z) s += part[z * n + e];
    out[e] = s;
  }
}

// Standalone per-frame argmax of z[f][0..J) (srp.py:74-80) into packed keys.
__global__ void __launch_bounds__(256)
argmax_kernel(const float* __restrict__ z, int64_t ldz, int64_t J, int64_t F,
              unsigned long long* __restrict__ keys) {
  const int64_t f = blockIdx.y;
  const float* row = z + f * ldz;
  unsigned long long key = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < J;
       i += (int64_t)gridDim.x * blockDim.x)
    key = key_max(key, make_key(__ldg(row + i), (uint32_t)i));
  key = warp_key_max(key);
  __shared__ unsigned long long red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) key = key_max(key, red[w]);
    key = key_max(key, red[0]);
    if (key) atomicMax(keys + f, key);
  }
}

__global__ void decode_keys_kernel(const unsigned long long* __restrict__ keys, int64_t F,
                                   int64_t* __restrict__ index, float* __restrict__ value) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const unsigned long long k = keys[f];
  const uint32_t hi = (uint32_t)(k >> 32);
  const uint32_t bits = (hi & 0x80000000u) ? (hi & 0x7FFFFFFFu) : ~hi;
  if (index) index[f] = (int64_t)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFu));
  if (value) value[f] = __uint_as_float(bits);
}

constexpr int kMaxSplit = 16;

// `split_ws` (nullable): kMaxSplit * F * I floats of scratch enabling split-K for
// small-output / long-K products (the low-rank factor products); out must then be
// dense (ldo == I) and keys unused.
int gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* out, int64_t ldo,
            int64_t I, int64_t F, int64_t K, float alpha, uint64_t* keys, cudaStream_t st,
            const char* what, bool b_trans = false, float* split_ws = nullptr) {
  if (I <= 0 || F <= 0) return SRPGPU_OK;
  const bool narrow = I <= 32;                       // 32 x 128 tiles (no half-empty 64-row tiles)
  const int64_t ti = narrow ? 32 : kGI, tf = 4096 / ti;
  const int64_t ctas = ((I + ti - 1) / ti) * ((F + tf - 1) / tf);
  int64_t split = 1;
  if (split_ws && !keys && ldo == I && ctas < 4 * num_sms())
    split = std::max<int64_t>(1, std::min<int64_t>({(int64_t)kMaxSplit, (4 * num_sms() + ctas - 1) / ctas,
                                                    K / 256}));
  const int64_t chunk = ((K + split - 1) / split + kGK - 1) / kGK * kGK;
  split = (K + chunk - 1) / chunk;
  SRPGPU_CHECK_ARG((I + ti - 1) / ti <= 65535, SRPGPU_ERR_DIMENSION, "%s: too many candidates", what);
  dim3 grid((unsigned)((F + tf - 1) / tf), (unsigned)((I + ti - 1) / ti), (unsigned)split);
  float* dst = split > 1 ? split_ws : out;
  const float a = split > 1 ? 1.0f : alpha;
  auto* kp = reinterpret_cast<unsigned long long*>(keys);
  if (b_trans) {
    if (narrow) gemm_nt_kernel<true, 32><<<grid, 256, 0, st>>>(A, lda, B, ldb, dst, ldo, I, F, K, a, kp, 0, chunk);
    else gemm_nt_kernel<true, 64><<<grid, 256, 0, st>>>(A, lda, B, ldb, dst, ldo, I, F, K, a, kp, 0, chunk);
  } else {
    if (narrow) gemm_nt_kernel<false, 32><<<grid, 256, 0, st>>>(A, lda, B, ldb, dst, ldo, I, F, K, a, kp, 0, chunk);
    else gemm_nt_kernel<false, 64><<<grid, 256, 0, st>>>(A, lda, B, ldb, dst, ldo, I, F, K, a, kp, 0, chunk);
  }
  SRPGPU_CHECK_LAUNCH(what);
  if (split > 1) {
    const int64_t n = F * I;
    splitk_reduce_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4 * num_sms()), 256, 0, st>>>(
        split_ws, split, n, out);
    SRPGPU_CHECK_LAUNCH(what);
    (void)alpha;   // alpha == 1 for the factor products that split
  }
  return SRPGPU_OK;
}

int reset_keys(uint64_t* keys, int64_t F, cudaStream_t st) {
  if (!keys || F <= 0) return SRPGPU_OK;
  if (cudaMemsetAsync(keys, 0, (size_t)F * sizeof(uint64_t), st) != cudaSuccess) {
    set_error("argmax key reset failed");
    return SRPGPU_ERR_LAUNCH;
  }
  return SRPGPU_OK;
}

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* out,
                              int64_t ldo, int64_t rows_i, int64_t rows_f, int64_t depth, float alpha,
                              uint64_t* keys, srpgpu_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, rows_f, st);
  if (s) return s;
  return gemm_nt(A, lda, B, ldb, out, ldo, rows_i, rows_f, depth, alpha, keys, st, "gemm_nt");
}

extern "C" int srpgpu_slri_map(const float* samples, int64_t samples_ld, int64_t num_frames,
                               int32_t total_samples,
                               const float* fat, const float* tall, int32_t rank,
                               int64_t num_candidates, float* work, float* z, uint64_t* keys,
                               srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rank >= 1, SRPGPU_ERR_VALUE, "slri_map: rank must be >= 1");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  // work[f][r] = sum_s fat[r][s] xi[s][f]   (samples lag-major [S][samples_ld]; 0 = frame-major)
  s = gemm_nt(fat, total_samples, samples, samples_ld ? samples_ld : total_samples, work, rank, rank,
              num_frames, total_samples, 1.0f, nullptr, st, "slri_map(fat)", samples_ld != 0,
              work + num_frames * (int64_t)rank);
  if (s) return s;
  return lowrank_out(tall, rank, work, rank, z, num_candidates, num_candidates, num_frames, rank, 1.0f,
                     keys, st, "slri_map(tall)");
}

// The rank-R candidate products on the tensor cores: the factor product work[F][R]
// (fp32 SIMT, as above) is split into bf16 hi/lo planes and z = tall . work^T runs on
// the dense-operand tcgen05 kernel of interp_tc.cu (K = R: the product is bound by the
// z write, not by the MMA).  tall_planes: [2][J][cols8] (srpgpu_split_bf16 of tall).
extern "C" int srpgpu_slri_map_tc(const float* samples, int64_t samples_ld, int64_t num_frames,
                                  int32_t total_samples, const float* fat, const void* tall_planes,
                                  int32_t rank, int32_t cols8, int64_t num_candidates, float* work,
                                  void* work_planes, float* z, uint64_t* keys, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rank >= 1 && cols8 >= rank && cols8 % 8 == 0, SRPGPU_ERR_VALUE,
                   "slri_map_tc: rank must be >= 1 and cols8 >= rank, a multiple of 8");
  cudaStream_t st = as_stream(stream);
  if (num_frames <= 0) return srpgpu_interp_map_tc(work_planes, 0, tall_planes, num_candidates, cols8, z, keys, stream);
  int s = gemm_nt(fat, total_samples, samples, samples_ld ? samples_ld : total_samples, work, rank, rank,
                  num_frames, total_samples, 1.0f, nullptr, st, "slri_map(fat)", samples_ld != 0,
                  work + num_frames * (int64_t)rank);
  if (s) return s;
  if ((s = srpgpu_split_bf16(work, rank, 0, num_frames, rank, work_planes, cols8, stream))) return s;
  return srpgpu_interp_map_tc(work_planes, num_frames, tall_planes, num_candidates, cols8, z, keys, stream);
}

// lr_map with the output product on the tensor cores; tall2_planes = split of
// [2 Re tall, -2 Im tall] ([2][J][cols8], cols8 >= 2R).
extern "C" int srpgpu_lr_map_tc(const float* gcc, int64_t num_frames, int32_t gcc_len, const float* fat2,
                                const void* tall2_planes, int32_t rank, int32_t cols8, int64_t num_candidates,
                                float* work, void* work_planes, float* z, uint64_t* keys,
                                srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rank >= 1 && cols8 >= 2 * rank && cols8 % 8 == 0, SRPGPU_ERR_VALUE,
                   "lr_map_tc: rank must be >= 1 and cols8 >= 2 rank, a multiple of 8");
  cudaStream_t st = as_stream(stream);
  if (num_frames <= 0) return srpgpu_interp_map_tc(work_planes, 0, tall2_planes, num_candidates, cols8, z, keys, stream);
  int s = gemm_nt(fat2, 2 * (int64_t)gcc_len, gcc, 2 * (int64_t)gcc_len, work, 2 * rank, 2 * rank, num_frames,
                  2 * (int64_t)gcc_len, 1.0f, nullptr, st, "lr_map(fat)", false,
                  work + num_frames * (int64_t)(2 * rank));
  if (s) return s;
  if ((s = srpgpu_split_bf16(work, 2 * rank, 0, num_frames, 2 * rank, work_planes, cols8, stream))) return s;
  return srpgpu_interp_map_tc(work_planes, num_frames, tall2_planes, num_candidates, cols8, z, keys, stream);
}

extern "C" int srpgpu_lr_map(const float* gcc, int64_t num_frames, int32_t gcc_len,
                             const float* fat2, const float* tall2, int32_t rank,
                             int64_t num_candidates, float* work, float* z, uint64_t* keys,
                             srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rank >= 1, SRPGPU_ERR_VALUE, "lr_map: rank must be >= 1");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  // work[f][0:R] = Re(fat psi_f), work[f][R:2R] = Im(fat psi_f); fat2 is (2R) x (2 PB)
  s = gemm_nt(fat2, 2 * (int64_t)gcc_len, gcc, 2 * (int64_t)gcc_len, work, 2 * rank, 2 * rank,
              num_frames, 2 * (int64_t)gcc_len, 1.0f, nullptr, st, "lr_map(fat)", false,
              work + num_frames * (int64_t)(2 * rank));
  if (s) return s;
  // z = [2 Re tall, -2 Im tall] . work
  return lowrank_out(tall2, 2 * rank, work, 2 * rank, z, num_candidates, num_candidates, num_frames,
                     2 * rank, 1.0f, keys, st, "lr_map(tall)");
}

extern "C" int srpgpu_srp_map_simt(const float* gcc, int64_t num_frames, int32_t gcc_len,
                                   const float* h2, int64_t num_candidates, float* z, uint64_t* keys,
                                   srpgpu_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  return gemm_nt(h2, 2 * (int64_t)gcc_len, gcc, 2 * (int64_t)gcc_len, z, num_candidates,
                 num_candidates, num_frames, 2 * (int64_t)gcc_len, 2.0f, keys, st, "srp_map(simt)");
}

extern "C" int srpgpu_argmax(const float* z, int64_t num_frames, int64_t num_candidates, int64_t ldz,
                             uint64_t* keys, srpgpu_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames <= 0 || num_candidates <= 0) return SRPGPU_OK;
  SRPGPU_CHECK_ARG(num_frames <= 65535, SRPGPU_ERR_DIMENSION, "argmax: too many frames per call");
  const int bx = (int)std::min<int64_t>((num_candidates + 255) / 256, 64);
  dim3 grid(bx, (unsigned)num_frames);
  argmax_kernel<<<grid, 256, 0, st>>>(z, ldz, num_candidates, num_frames,
                                      reinterpret_cast<unsigned long long*>(keys));
  SRPGPU_CHECK_LAUNCH("argmax");
  return SRPGPU_OK;
}

extern "C" int srpgpu_decode_keys(const uint64_t* keys, int64_t num_frames, int64_t* index,
                                  float* value, srpgpu_stream_t stream) {
  if (num_frames <= 0) return SRPGPU_OK;
  decode_keys_kernel<<<(unsigned)((num_frames + 255) / 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const unsigned long long*>(keys), num_frames, index, value);
  SRPGPU_CHECK_LAUNCH("decode_keys");
  return SRPGPU_OK;
}
