// Sparse interpolation map (SSPI-SRP) on sm_100a:
//   z[f][i] = sum_p sum_{kept (i,p,n)} Lambda[i][p,n] * xi[(p,n)][f]
// restating interpolation.py:188-195 (_dot_sparse_rows :121-126).  With a keep-all
// operator the same kernel is si_map (:129-136), so sspi(all) == si bit-for-bit as in
// the reference (interpolation.py:112-126).
//
// Operator layout: "tiled band" (built once on the host from the reference CSR).
// Candidates are cut into groups of 4 consecutive rows, placed 8 to a tile (in index
// order by default; any permutation of the groups is allowed -- BandOperator in maps.py).
// For every (group, pair) the union of the lags kept by the group's 4 candidates
// becomes a run of records {u32 sample index, 3 x pad, f32 weight[4]} (weight 0
// where a candidate does not keep that lag).  A tile's blob is contiguous:
//     meta[32] : u32 start record of slots 0..7, meta[8] = record total,
//                meta[16 + g] = first candidate of slot g, meta[24 + g] = its count
//     records  : slot 0 (pairs ascending, then sample index), slot 1, ...
// so each warp walks one flat record range, and one TMA bulk copy stages the tile
// (or, for large tiles, warps read their records from global memory).
//
// Samples are lag-major xi[s][f] (row pitch ld, frames contiguous).  CTA = 32
// candidates x (n x 128) frames: the operator tile is staged once, then the CTA
// walks its frame tiles.  Lane = 4 consecutive frames, warp = one group of 4
// candidates.  Per record: one broadcast shared-memory read (index + 4 weights), one
// coalesced 16-byte L1 read of xi[s][f..f+3], 16 FMAs into registers -- the xi value is
// reused from registers by the group's 4 candidates.  z is stored straight from
// registers (16-byte streaming stores when rows are aligned); the per-frame argmax
// is reduced in registers (4 candidates), across warps in shared memory, and
// folded into packed 64-bit keys with one atomicMax per frame per CTA.
#include "common.cuh"

namespace srpgpu {

constexpr int kWarps = 8;
constexpr int kGroup = 4;                          // candidates per warp
constexpr int kTileI = kWarps * kGroup;            // 32 candidates per CTA
constexpr int kTileF = 128;                        // frames per frame tile (4 per lane)
constexpr int64_t kStageMax = 64 * 1024;          // max bytes of a staged operator tile
constexpr int kMetaBytes = 128;

struct __align__(16) BandRec {
  uint32_t s, pad0, pad1, pad2;
  float4 w;
};

struct BandParams {
  const float* xi;            // [S][ld]
  int64_t ld;
  int64_t F;
  int32_t S;
  int32_t P;
  const int64_t* tile_off;    // [T+1] byte offsets of the tile blobs
  const unsigned char* blob;
  int64_t J;
  float* z;                   // [F][J] or null
  unsigned long long* keys;   // [F] or null
  int32_t rec_cap;            // records per staged chunk
  int32_t ftiles_per_cta;     // frame tiles walked by one CTA
};

__device__ __forceinline__ uint32_t s_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s_addr(dst)),
      "l"(src), "r"(bytes), "r"(s_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(s_addr(bar)),
      "r"(phase)
      : "memory");
}

// Direct variant: records read from global memory, software-pipelined one group of 4
// ahead so that only the xi load latency is exposed (records do not depend on data).
__device__ __forceinline__ void accumulate_direct(float (&acc)[kGroup][4], const BandRec* rr, int n,
                                                  const float* xcol, int64_t ld) {
  constexpr int U = 4;
  uint32_t s[U];
  float4 w[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    s[u] = u < n ? __ldg(&rr[u].s) : 0u;
    w[u] = u < n ? __ldg(&rr[u].w) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int r = 0; r < n; r += U) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)   // padding slots read row 0 with zero weights
      x[u] = __ldg(reinterpret_cast<const float4*>(xcol + (int64_t)s[u] * ld));
    uint32_t sn[U];
    float4 wn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = r + U + u;
      sn[u] = q < n ? __ldg(&rr[q].s) : 0u;
      wn[u] = q < n ? __ldg(&rr[q].w) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[0][0] = fmaf(w[u].x, x[u].x, acc[0][0]); acc[0][1] = fmaf(w[u].x, x[u].y, acc[0][1]);
      acc[0][2] = fmaf(w[u].x, x[u].z, acc[0][2]); acc[0][3] = fmaf(w[u].x, x[u].w, acc[0][3]);
      acc[1][0] = fmaf(w[u].y, x[u].x, acc[1][0]); acc[1][1] = fmaf(w[u].y, x[u].y, acc[1][1]);
      acc[1][2] = fmaf(w[u].y, x[u].z, acc[1][2]); acc[1][3] = fmaf(w[u].y, x[u].w, acc[1][3]);
      acc[2][0] = fmaf(w[u].z, x[u].x, acc[2][0]); acc[2][1] = fmaf(w[u].z, x[u].y, acc[2][1]);
      acc[2][2] = fmaf(w[u].z, x[u].z, acc[2][2]); acc[2][3] = fmaf(w[u].z, x[u].w, acc[2][3]);
      acc[3][0] = fmaf(w[u].w, x[u].x, acc[3][0]); acc[3][1] = fmaf(w[u].w, x[u].y, acc[3][1]);
      acc[3][2] = fmaf(w[u].w, x[u].z, acc[3][2]); acc[3][3] = fmaf(w[u].w, x[u].w, acc[3][3]);
      s[u] = sn[u];
      w[u] = wn[u];
    }
  }
}

template <bool kGlobal>
__device__ __forceinline__ void accumulate(float (&acc)[kGroup][4], const BandRec* rr, int n,
                                           const float* xcol, int64_t ld) {
#pragma unroll 4
  for (int r = 0; r < n; ++r) {
    uint32_t s;
    float4 w;
    if (kGlobal) {   // uniform address across the warp: one broadcast read-only load
      s = __ldg(&rr[r].s);
      w = __ldg(&rr[r].w);
    } else {
      s = rr[r].s;
      w = rr[r].w;
    }
    const float4 x = __ldg(reinterpret_cast<const float4*>(xcol + (int64_t)s * ld));
    acc[0][0] = fmaf(w.x, x.x, acc[0][0]); acc[0][1] = fmaf(w.x, x.y, acc[0][1]);
    acc[0][2] = fmaf(w.x, x.z, acc[0][2]); acc[0][3] = fmaf(w.x, x.w, acc[0][3]);
    acc[1][0] = fmaf(w.y, x.x, acc[1][0]); acc[1][1] = fmaf(w.y, x.y, acc[1][1]);
    acc[1][2] = fmaf(w.y, x.z, acc[1][2]); acc[1][3] = fmaf(w.y, x.w, acc[1][3]);
    acc[2][0] = fmaf(w.z, x.x, acc[2][0]); acc[2][1] = fmaf(w.z, x.y, acc[2][1]);
    acc[2][2] = fmaf(w.z, x.z, acc[2][2]); acc[2][3] = fmaf(w.z, x.w, acc[2][3]);
    acc[3][0] = fmaf(w.w, x.x, acc[3][0]); acc[3][1] = fmaf(w.w, x.y, acc[3][1]);
    acc[3][2] = fmaf(w.w, x.z, acc[3][2]); acc[3][3] = fmaf(w.w, x.w, acc[3][3]);
  }
}

// kDirect: records are read by each warp straight from global memory (L1/L2, broadcast)
// instead of being staged in shared memory -- for operator tiles too large to stage
// without dropping to one CTA per SM (cfg4: ~146 KB per tile).  No CTA barrier in the
// accumulation loop; ~25 KB of shared memory per CTA, so occupancy is register-bound.
template <bool kDirect>
__global__ void __launch_bounds__(kWarps * 32)
sspi_band_kernel(const BandParams prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t meta[32];
  unsigned long long* kred = reinterpret_cast<unsigned long long*>(smem_raw);        // [TF][8]
  float* zs = reinterpret_cast<float*>(smem_raw + (size_t)kTileF * kWarps * 8);      // [TF][TI+1]
  BandRec* recs = reinterpret_cast<BandRec*>(smem_raw + (size_t)kTileF * kWarps * 8 +
                                             (size_t)kTileF * (kTileI + 1) * 4);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = blockIdx.x;
  const unsigned char* tb = prm.blob + prm.tile_off[tile];
  const uint32_t tile_bytes = (uint32_t)(prm.tile_off[tile + 1] - prm.tile_off[tile]);
  const BandRec* grec = reinterpret_cast<const BandRec*>(tb + kMetaBytes);

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) meta[tid] = reinterpret_cast<const uint32_t*>(tb)[tid];
  __syncthreads();
  const uint32_t total = meta[8];
  const uint32_t g0 = meta[warp], g1 = (warp + 1 < kWarps) ? meta[warp + 1] : total;
  const bool whole = kDirect || total <= (uint32_t)prm.rec_cap;
  uint32_t phase = 0;
  if (!kDirect && whole && total > 0) {   // one TMA bulk copy for the whole operator tile, reused by all frame tiles
    if (tid == 0) {
      mbar_arm(&bar, tile_bytes - kMetaBytes);
      bulk_copy(recs, grec, tile_bytes - kMetaBytes, &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
  }

  const int64_t ftile0 = (int64_t)blockIdx.y * prm.ftiles_per_cta;
  for (int64_t ft = ftile0; ft < ftile0 + prm.ftiles_per_cta; ++ft) {
    const int64_t f0 = ft * kTileF;
    if (f0 >= prm.F) break;
    float acc[kGroup][4];
#pragma unroll
    for (int c = 0; c < kGroup; ++c)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[c][t] = 0.f;
    const int64_t fl = f0 + 4 * lane;
    const bool lane_ok = fl < prm.ld;
    const float* xcol = prm.xi + fl;
    if (kDirect) {
      if (lane_ok) accumulate_direct(acc, grec + g0, (int)(g1 - g0), xcol, prm.ld);
    } else if (whole) {
      if (lane_ok) accumulate<false>(acc, recs + g0, (int)(g1 - g0), xcol, prm.ld);
    } else {
      for (uint32_t c0 = 0; c0 < total; c0 += (uint32_t)prm.rec_cap) {
        const uint32_t c1 = min(total, c0 + (uint32_t)prm.rec_cap);
        __syncthreads();   // previous chunk fully consumed
        if (tid == 0) {
          mbar_arm(&bar, (c1 - c0) * (uint32_t)sizeof(BandRec));
          bulk_copy(recs, grec + c0, (c1 - c0) * (uint32_t)sizeof(BandRec), &bar);
        }
        mbar_wait(&bar, phase);
        phase ^= 1u;
        const uint32_t a = max(g0, c0), b = min(g1, c1);
        if (lane_ok && b > a) accumulate<false>(acc, recs + (a - c0), (int)(b - a), xcol, prm.ld);
      }
    }

    // ---- outputs: z from registers, per-frame argmax keys
    const int64_t ib = meta[16 + warp];                 // the slot's group: first candidate, count
    const int nvalid = (int)meta[24 + warp];
    const bool aligned = (prm.J % 4 == 0);
    if (kDirect) {   // warps finish independently: no CTA barrier, one atomic per (lane, frame)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int64_t f = fl + t;
        if (f >= prm.F || nvalid == 0) continue;
        float best = acc[0][t];
        int bi = 0;
#pragma unroll
        for (int c = 1; c < kGroup; ++c)
          if (c < nvalid && acc[c][t] > best) { best = acc[c][t]; bi = c; }
        if (prm.z) {
          float* zr = prm.z + f * prm.J + ib;
          if (aligned && nvalid == kGroup) {
            __stcs(reinterpret_cast<float4*>(zr), make_float4(acc[0][t], acc[1][t], acc[2][t], acc[3][t]));
          } else {
#pragma unroll
            for (int c = 0; c < kGroup; ++c)
              if (c < nvalid) __stcs(zr + c, acc[c][t]);
          }
        }
        if (prm.keys) atomicMax(prm.keys + f, make_key(best, (uint32_t)(ib + bi)));
      }
      continue;
    }
    const bool vec = prm.z && nvalid == kGroup && aligned;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t f = fl + t;
      unsigned long long key = 0ull;
      if (f < prm.F && nvalid > 0) {
        float best = acc[0][t];
        int bi = 0;
#pragma unroll
        for (int c = 1; c < kGroup; ++c)
          if (c < nvalid && acc[c][t] > best) { best = acc[c][t]; bi = c; }
        key = make_key(best, (uint32_t)(ib + bi));
        if (vec)   // 16-byte rows: store straight from registers
          __stcs(reinterpret_cast<float4*>(prm.z + f * prm.J + ib),
                 make_float4(acc[0][t], acc[1][t], acc[2][t], acc[3][t]));
      }
      kred[(4 * lane + t) * kWarps + warp] = key;
      if (prm.z && !aligned) {
#pragma unroll
        for (int c = 0; c < kGroup; ++c) zs[(4 * lane + t) * (kTileI + 1) + warp * kGroup + c] = acc[c][t];
      }
    }
    __syncthreads();
    if (prm.z && !aligned) {   // unaligned rows: transpose through shared memory, coalesced rows
      const int slot = lane >> 2, c = lane & 3;          // column lane = slot * 4 + c
      const bool live = c < (int)meta[24 + slot];
      const int64_t col = (int64_t)meta[16 + slot] + c;
      for (int row = warp; row < kTileF; row += kWarps) {
        const int64_t fg = f0 + row;
        if (fg >= prm.F) break;
        if (live) prm.z[fg * prm.J + col] = zs[row * (kTileI + 1) + lane];
      }
    }
    if (prm.keys && tid < kTileF) {
      const int64_t f = f0 + tid;
      if (f < prm.F) {
        unsigned long long k = kred[tid * kWarps];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) k = key_max(k, kred[tid * kWarps + w]);
        if (k) atomicMax(prm.keys + f, k);
      }
    }
    __syncthreads();   // kred reused by the next frame tile
  }
}

// Small-frame-count path (e.g. the per-frame reference call): a thread per
// (candidate, frame) walking its group's records in the tile kernel's order, so
// both kernels give bit-identical maps.
__global__ void sspi_band_rows_kernel(const BandParams prm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // operator position
  const int64_t f = blockIdx.y;
  const int64_t tile = t / kTileI;
  const int g = (int)((t % kTileI) / kGroup), c = (int)(t % kGroup);
  const int64_t tiles = (prm.J + kTileI - 1) / kTileI;
  bool live = tile < tiles;
  int64_t gi = 0;
  float acc = 0.f;
  if (live) {
    const unsigned char* tb = prm.blob + prm.tile_off[tile];
    const uint32_t* meta = reinterpret_cast<const uint32_t*>(tb);
    live = c < (int)meta[24 + g];
    gi = (int64_t)meta[16 + g] + c;
    if (live) {
      const BandRec* grec = reinterpret_cast<const BandRec*>(tb + kMetaBytes);
      const uint32_t r1 = (g + 1 < kWarps) ? meta[g + 1] : meta[8];
      for (uint32_t r = meta[g]; r < r1; ++r) {
        const float4 w = grec[r].w;
        const float wc = c == 0 ? w.x : c == 1 ? w.y : c == 2 ? w.z : w.w;
        acc = fmaf(wc, __ldg(prm.xi + (int64_t)grec[r].s * prm.ld + f), acc);
      }
      if (prm.z) prm.z[f * prm.J + gi] = acc;
    }
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
                               int32_t total_samples, int32_t num_pairs, const int64_t* tile_offsets,
                               const void* blob, int64_t num_candidates, int64_t max_pair_records,
                               int64_t max_tile_records, float* z, uint64_t* keys,
                               srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_pairs >= 1 && num_candidates >= 1 && total_samples >= 1, SRPGPU_ERR_DIMENSION,
                   "sspi_map: empty operator");
  SRPGPU_CHECK_ARG(num_candidates < 0xFFFFFFFFll, SRPGPU_ERR_DIMENSION, "sspi_map: too many candidates");
  SRPGPU_CHECK_ARG(samples_ld >= num_frames && samples_ld % 4 == 0, SRPGPU_ERR_VALUE,
                   "sspi_map: lag-major pitch must cover the frames and be a multiple of 4");
  SRPGPU_CHECK_ARG(((uintptr_t)samples & 15) == 0 && ((uintptr_t)blob & 15) == 0, SRPGPU_ERR_VALUE,
                   "sspi_map: operands must be 16-byte aligned");
  if (num_frames <= 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  BandParams prm = {};
  prm.xi = samples; prm.ld = samples_ld; prm.F = num_frames; prm.S = total_samples; prm.P = num_pairs;
  prm.tile_off = tile_offsets; prm.blob = reinterpret_cast<const unsigned char*>(blob);
  prm.J = num_candidates; prm.z = z; prm.keys = reinterpret_cast<unsigned long long*>(keys);
  if (keys) {
    if (cudaMemsetAsync(keys, 0, (size_t)num_frames * sizeof(uint64_t), st) != cudaSuccess) {
      set_error("sspi_map: key reset failed");
      return SRPGPU_ERR_LAUNCH;
    }
  }
  if (num_frames < 32) {
    const int64_t slots = (num_candidates + kTileI - 1) / kTileI * kTileI;
    dim3 grid((unsigned)((slots + 255) / 256), (unsigned)num_frames);
    sspi_band_rows_kernel<<<grid, 256, 0, st>>>(prm);
    SRPGPU_CHECK_LAUNCH("sspi_map(rows)");
    return SRPGPU_OK;
  }
  // operator tiles up to kStageMax bytes are staged whole in shared memory (one bulk copy,
  // reused by every frame tile); larger tiles are read by each warp from global memory
  // (cfg2/cfg3 tiles: 6-18 KB, staged; cfg4: up to 143 KB, direct -- 2.2x faster there)
  const bool direct = max_tile_records * (int64_t)sizeof(BandRec) > kStageMax;
  (void)max_pair_records;
  prm.rec_cap = (int32_t)std::max<int64_t>(1, direct ? 1 : max_tile_records);
  const size_t smem = direct ? 0 : (size_t)kTileF * kWarps * 8 + (size_t)kTileF * (kTileI + 1) * 4 +
                                     (size_t)prm.rec_cap * sizeof(BandRec);
  auto kern = direct ? sspi_band_kernel<true> : sspi_band_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("sspi_map: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  const int64_t ctiles = (num_candidates + kTileI - 1) / kTileI;
  const int64_t ftiles = (num_frames + kTileF - 1) / kTileF;
  // walk several frame tiles per CTA (operator staged once) while keeping >= ~8 CTAs per SM
  int64_t per = std::max<int64_t>(1, std::min<int64_t>(8, (ctiles * ftiles) / (8 * (int64_t)num_sms())));
  prm.ftiles_per_cta = (int32_t)per;
  const int64_t gy = (ftiles + per - 1) / per;
  SRPGPU_CHECK_ARG(gy <= 65535, SRPGPU_ERR_DIMENSION, "sspi_map: too many frames per call");
  dim3 grid((unsigned)ctiles, (unsigned)gy);
  kern<<<grid, kWarps * 32, smem, st>>>(prm);
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
