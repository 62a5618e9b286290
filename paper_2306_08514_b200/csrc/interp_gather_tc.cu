// SSPI / SI on the tensor cores for long sample vectors (BASELINE cfg4: S = 7028 lags):
// per-tile gathered lag windows (layout built on the host by tiles.py).
//
//   z[f][j] = sum_s Lambda[j][s] xi[f][s]      interpolation.py:121-126, 188-195
//
// Candidates come in tiles of 256 that are compact in TDOA space; a tile's operator is
// dense over K = its candidates' kept lag windows (pair by pair, rounded up to groups of
// 8 lags), stored in 64-lag blocks of two 128-row slabs (bf16 hi / lo planes).  The
// matching samples are gathered from lag-major, natural-lag-order xi planes [S][F8]
// (frames contiguous): a group is 8 lag rows, loaded as four 128-byte-swizzled TMA boxes
// of 64 frames x 8 lags.  Each gathered sample stage feeds both 128-row halves of the
// tile (two MMAs per step), which halves the gather TMA traffic per flop: with 128-row
// tiles the kernel was bound by the TMA box rate (measured: a quarter of the boxes for
// the same MMA work ran 2x faster).  A frame-major gather would need one 16-byte box per
// (frame, group) row: 6x slower again.
//
// D_h = A_h . B^T per half h: A_h = slab (M = 128 candidates = TMEM lanes, K-major,
// 64-byte swizzle, 32-lag k-blocks), B = gathered xi (N = 256 frames = TMEM columns,
// MN-major, 128-byte swizzle: 1 KB atoms of 64 frames x 8 lags, 1 KB apart along N (LBO)
// and 4 KB apart along K (SBO)).  Three kind::f16 MMAs per 16-lag step (bf16 hi/lo split,
// as interp_tc.cu); the two halves fill the 512 TMEM columns.  Persistent CTAs take the
// work units (frame-tile group, tile, frame tile) round-robin.
// Roles: warp 0 TMA producer (lanes 0-7 one plane x group each, 8-11 the slabs), warp 1
// TMEM allocator + MMA issuer, warps 2-9 epilogue (lane quarter warp % 4 of one half):
// the map goes out in tile order, 128 contiguous bytes per warp store (a gather pass
// restores grid order: scattered 4-byte stores made the L2 read-modify-write each
// sector), and the per-frame argmax is a butterfly max across the lanes plus a ballot
// for the lowest winning candidate (tile rows are ascending).
#include <cstdlib>
#include <cuda_bf16.h>

#include "tc_common.cuh"

namespace srpgpu {
namespace gtc {

using namespace tc;

constexpr int GM = 128;   // candidates per tile half (TMEM lanes)
constexpr int GT = 256;   // candidates per tile (two halves)
constexpr int GN = 256;   // frames per unit
constexpr int GB = 64;    // lags per operator block (slab width)
constexpr int GK = 32;    // lags per pipeline stage
constexpr int GG = 8;     // lags per gathered group (8 rows of the lag-major samples)
constexpr int GA = 64;    // frames per MN atom (128 bytes)
constexpr int NG = GK / GG;          // groups per stage
constexpr int UK = 16;    // kind::f16 MMA K
constexpr int NS = 3;     // operand stages (64 KB each)
constexpr int kEpi = 8;
constexpr int kThreads = 32 * (2 + kEpi);
constexpr int FG = 8;     // frame tiles per unit group
constexpr int kMaxBlocks = 128;                   // 64-lag blocks per tile (K <= 8192 lags)
constexpr int kMaxGroups = kMaxBlocks * (GB / GG);

struct __align__(1024) Smem {
  uint16_t a[NS][2][2][GM * GK];       // [half][plane] slab columns (8 KB each, 64-byte swizzle)
  uint16_t b[NS][2][NG][GN * GG];      // [plane][group] 4 atoms [8 lags][64 frames] (4 KB each)
  int32_t rows[2][kMaxGroups];         // the current / next unit's group rows (producer only)
  uint64_t full[NS], empty[NS], tfull, tempty;
  uint32_t tmem_base;
};

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// MN-major operand, 128-byte swizzle: 1 KB atoms (8 K rows x 64 MN elements);
// LBO = distance between MN-adjacent atoms, SBO = between K-adjacent 8-row groups
__device__ __forceinline__ uint64_t desc_mn128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)(1024 >> 4) << 16;             // LBO: next 64 frames
  d |= (uint64_t)((GN * GG * 2) >> 4) << 32;    // SBO: next 8-lag group (4 KB)
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

struct Unit {
  int t, n;
};

__device__ __forceinline__ bool decode(int u, int T, int n_tiles, Unit& out) {
  const int per = T * FG;
  const int g = u / per, rem = u - g * per;
  out.t = rem / FG;
  out.n = g * FG + (rem - out.t * FG);
  return out.n < n_tiles;
}

// Epilogue warps (2 + 4 * half + quarter): per unit, wait for the accumulator, drain the
// warp's TMEM lane quarter of its tile half 32 frames at a time, store the map (tile order
// or grid order) and fold the per-frame argmax (butterfly max across the lanes + a ballot
// for the lowest winning candidate: tile rows are ascending); then free the accumulator.
__device__ __forceinline__ void epilogue(uint32_t tmem, int warp, int lane, int64_t F, int64_t J, int32_t T,
                                         int n_tiles, int u_total, uint64_t* tfull, uint64_t* tempty,
                                         const int32_t* __restrict__ tile_rows, float* __restrict__ zt,
                                         float* __restrict__ zg, unsigned long long* __restrict__ keys) {
  const int q = warp & 3;                          // TMEM lane quarter this warp may access
  const int half = (warp - 2) >> 2;                // which tile half (TMEM columns half * 256)
  const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * GN);
  const int64_t ldt = (int64_t)T * GT;
  uint32_t it = 0;
  for (int u = blockIdx.x; u < u_total; u += gridDim.x) {
    Unit w;
    if (!decode(u, T, n_tiles, w)) continue;
    const int r = half * GM + q * 32 + lane;         // tile row
    const int jrow = __ldg(tile_rows + (int64_t)w.t * GT + r);   // -1: padding row
    mbar_wait(tfull, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool any = __any_sync(0xffffffffu, jrow >= 0);
#pragma unroll 1
    for (int c = 0; c < GN / 32; ++c) {
      uint32_t rr[32];
      tmem_ld32(lane_base + c * 32, rr);
      const int64_t f0 = (int64_t)w.n * GN + c * 32;
      if (f0 >= F || !any) continue;               // warp-uniform (after the aligned load)
      if (zg) {   // grid order: the tile's rows are ascending candidates (runs of neighbours)
        if (jrow >= 0) {
          float* zc = zg + f0 * J + jrow;
          if (f0 + 32 <= F) {
#pragma unroll
            for (int t = 0; t < 32; ++t) __stcs(zc + t * J, __uint_as_float(rr[t]));
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (f0 + t < F) __stcs(zc + t * J, __uint_as_float(rr[t]));
          }
        }
      } else if (zt) {   // tile order: a warp's 32 rows are 128 contiguous bytes of the frame's row
        float* zc = zt + f0 * ldt + (int64_t)w.t * GT + r;
        if (f0 + 32 <= F) {
#pragma unroll
          for (int t = 0; t < 32; ++t) __stcs(zc + t * ldt, __uint_as_float(rr[t]));
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (f0 + t < F) __stcs(zc + t * ldt, __uint_as_float(rr[t]));
        }
      }
      if (keys) {
        uint32_t ob[32], v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = ob[t] = jrow >= 0 ? ordered_bits(__uint_as_float(rr[t])) : 0u;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int t = 0; t < o; ++t) {
            const uint32_t send = up ? v[t] : v[t + o];
            const uint32_t keep = up ? v[t + o] : v[t];
            v[t] = max(keep, __shfl_xor_sync(0xffffffffu, send, o));
          }
        }
        // lane t holds frame f0 + t's maximum in v[0]; the lowest lane (= lowest candidate) wins
        uint32_t win = 0;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const uint32_t vt = __shfl_sync(0xffffffffu, v[0], t);
          const uint32_t m = __ballot_sync(0xffffffffu, ob[t] == vt);
          if (lane == t) win = (uint32_t)(__ffs(m) - 1);
        }
        const int jw = __shfl_sync(0xffffffffu, jrow, (int)win);
        if (f0 + lane < F && v[0] != 0u)
          atomicMax(keys + f0 + lane,
                    ((unsigned long long)v[0] << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)jw));
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
    ++it;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
gather_tc_kernel(const __grid_constant__ CUtensorMap ma_hi, const __grid_constant__ CUtensorMap ma_lo,
                 const __grid_constant__ CUtensorMap mb_hi, const __grid_constant__ CUtensorMap mb_lo, int64_t F,
                 int64_t J, int32_t T, const int32_t* __restrict__ group_col, const int32_t* __restrict__ tile_blk,
                 const int32_t* __restrict__ tile_nkb, const int32_t* __restrict__ tile_rows,
                 float* __restrict__ zt, float* __restrict__ zg, unsigned long long* __restrict__ keys) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)((F + GN - 1) / GN);
  // units round-robin over the CTAs: at any moment the grid works on ~gridDim.x consecutive
  // units of ONE frame-tile group, so that group's xi columns stay L2-resident and each
  // tile's slabs are fetched from DRAM once per group (the FG CTAs sharing them run together)
  const int u_total = ((n_tiles + FG - 1) / FG) * T * FG;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ma_hi);
    prefetch_tmap(&ma_lo);
    prefetch_tmap(&mb_hi);
    prefetch_tmap(&mb_lo);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tfull, 1);
    mbar_init(&sm.tempty, kEpi);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // the unit's group rows are staged in shared memory (one coalesced load per unit,
    // prefetched a unit ahead) so the per-stage loop has no dependent global load;
    // lane 0 waits and arms the stage; lanes 0-7 then each load one (plane, group):
    // four 64-frame atoms of its 8 lag rows; lanes 8-11 load the (half, plane) slabs
    constexpr uint32_t kBytes = 2u * (2 * GM * GK + GN * GK) * sizeof(uint16_t);
    const int plane = (lane >> 2) & 1, grp = lane & 3;
    const int ah = ((lane - 8) >> 1) & 1, ap = (lane - 8) & 1;
    const uint64_t keep = policy_evict_last();   // a tile's slabs are re-read for FG frame tiles
    auto next_unit = [&](int u, Unit& w) {
      while (u < u_total && !decode(u, T, n_tiles, w)) u += gridDim.x;
      return u;
    };
    auto stage_rows = [&](int buf, const Unit& w) {
      const int b0 = __ldg(tile_blk + w.t), nk = __ldg(tile_nkb + w.t);
      for (int i = lane; i < nk * (GB / GG); i += 32) sm.rows[buf][i] = __ldg(group_col + b0 * (GB / GG) + i);
    };
    uint32_t g = 0;
    int buf = 0;
    Unit w;
    int u = next_unit(blockIdx.x, w);
    if (u < u_total) stage_rows(0, w);
    while (u < u_total) {
      Unit wn;
      const int un = next_unit(u + gridDim.x, wn);
      if (un < u_total) stage_rows(buf ^ 1, wn);        // prefetch the next unit's rows
      __syncwarp();
      const int b0 = __ldg(tile_blk + w.t), nk = __ldg(tile_nkb + w.t);
      for (int kq = 0; kq < 2 * nk; ++kq, ++g) {       // 32-lag stages: half a block each
        const int blk = b0 + (kq >> 1), sub = kq & 1;
        const int row = sm.rows[buf][kq * NG + grp];
        const int s = g % NS;
        if (lane == 0) {
          mbar_wait(&sm.empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&sm.full[s], kBytes);
        }
        __syncwarp();
        if (lane < 8) {
          const CUtensorMap* mb = plane ? &mb_lo : &mb_hi;
#pragma unroll
          for (int a = 0; a < GN / GA; ++a)
            tma_load_2d(sm.b[s][plane][grp] + a * GA * GG, mb, &sm.full[s], w.n * GN + a * GA, row);
        } else if (lane < 12) {
          tma_load_2d_hint(sm.a[s][ah][ap], ap ? &ma_lo : &ma_hi, &sm.full[s], sub * GK, (2 * blk + ah) * GM, keep);
        }
      }
      __syncwarp();
      buf ^= 1;
      u = un;
      w = wn;
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // D f32, A/B bf16, A K-major, B MN-major (bit 16), N = 256, M = 128
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(GN >> 3) << 17) |
                                 ((uint32_t)(GM >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int u = blockIdx.x; u < u_total; u += gridDim.x) {
        Unit w;
        if (!decode(u, T, n_tiles, w)) continue;
        const int nk = __ldg(tile_nkb + w.t);
        mbar_wait(&sm.tempty, (it & 1) ^ 1);            // the previous unit's maps are drained
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kq = 0; kq < 2 * nk; ++kq, ++g) {
          const int s = g % NS;
          mbar_wait(&sm.full[s], (g / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int k = 0; k < GK / UK; ++k) {
            const uint64_t aoff = (uint64_t)((k * UK * 2) >> 4);
            const uint64_t bh = desc_mn128(sm.b[s][0][2 * k]), bl = desc_mn128(sm.b[s][1][2 * k]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t d = tmem + h * GN;
              const uint64_t a_h = smem_desc_sw64(sm.a[s][h][0]) + aoff, a_l = smem_desc_sw64(sm.a[s][h][1]) + aoff;
              mma_bf16(d, a_h, bh, idesc, (kq | k) != 0);
              mma_bf16(d, a_h, bl, idesc, 1u);
              mma_bf16(d, a_l, bh, idesc, 1u);
            }
          }
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull);
        ++it;
      }
    }
  } else {
    epilogue(tmem, warp, lane, F, J, T, n_tiles, u_total, &sm.tfull, &sm.tempty, tile_rows, zt, zg, keys);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// ---- 3xTF32 variant with fp32 chunk folds (FP32-class) -------------------------------
// Operands hi = tf32_rne(x), lo = tf32_rne(x - hi) (21+ significant bits; the lo.lo term
// is dropped).  The tensor pipe's own accumulation is not IEEE fp32: its error grows with
// the number of MMAs accumulated into one TMEM tile (measured ~1.6e-8 of max|z| per MMA
// step: 7.3e-6 at cfg4 with whole-tile accumulation), so the MMAs accumulate a CHUNK of
// CH stages (CH * 2 K steps x 3 passes) into one of two TMEM buffers and the epilogue
// warps fold each finished chunk into fp32 registers (round-to-nearest adds) while the
// MMAs fill the other buffer.  Two buffers x two tile halves fit the 512 TMEM columns
// with units of 128 frames (N = 128).
//   stage = 16 lags: A (slab) per half and plane 128 rows x 16 lags fp32 (64-byte rows,
//     64-byte swizzle, 8 KB); B (gathered xi) per plane and group 4 frame blocks of
//     [8 lags][32 frames] fp32 (1 KB each = two 512-byte atoms of the 32-byte-granular
//     128-byte swizzle MN-major tf32 requires), all 4 fetched by ONE 3D TMA box
//     {32 frames, 8 lags, 4 frame blocks} over the lag-major planes viewed as
//     {32, lags, frames / 32} (fallback: four 2D boxes when the 3D view cannot be encoded).
namespace g32 {
__device__ __forceinline__ void named_barrier(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int GK = 16;               // lags per stage
constexpr int GG = 4;                // lags per gathered group (one 4-row MN atom of the tf32 layout)
constexpr int NG = GK / GG;          // groups per stage
constexpr int kMaxGroups = kMaxBlocks * (GB / GG);
constexpr int GN = 128;              // frames per unit
constexpr int GA = 32;               // frames per frame block (128 bytes of fp32)
constexpr int NA = GN / GA;          // frame blocks per group
constexpr int UK = 8;                // kind::tf32 MMA K
constexpr int NS = 4;                // operand stages (48 KB each)

struct __align__(1024) Smem {
  float b[NS][2][NG][GN * GG];       // [plane][group] 4 frame blocks of [4 lags][32 frames] (2 KB)
  float a[NS][2][2][GM * GK];        // [half][plane] slab columns (8 KB)
  int32_t rows[2][kMaxGroups];
  uint64_t full[NS], empty[NS], tfull[2], tempty[2];
  uint32_t tmem_base;
};

// units (frame-tile group of fg frame tiles, tile, frame tile), frame tile fastest: the
// group's gathered samples stay L2-resident while every tile's slabs stream through once
__device__ __forceinline__ bool decode32(int u, int T, int fg, int n_tiles, Unit& out) {
  const int per = T * fg;
  const int g = u / per, rem = u - g * per;
  out.t = rem / fg;
  out.n = g * fg + (rem - out.t * fg);
  return out.n < n_tiles;
}

// Unit order of the pair kernel with tile chunks (tc > 0): chunk of tc tiles, frame group, tile
// of the chunk, frame tile of the group -- a chunk's slabs stay in L2 (evict_last) while every
// frame group streams past them, so each slab comes from DRAM once per launch instead of once
// per group.  tc == 0: group, tile, frame tile (decode32).
__device__ __forceinline__ bool decode_pair(int u, int T, int fg, int n_tiles, int tc, Unit& out) {
  if (tc <= 0) return decode32(u, T, fg, n_tiles, out);
  const int ng = (n_tiles + fg - 1) / fg;
  const int per_g = tc * fg, per_c = ng * per_g;
  const int c = u / per_c, r = u - c * per_c;
  const int g = r / per_g, r2 = r - g * per_g;
  const int tl = r2 / fg;
  out.t = c * tc + tl;
  out.n = g * fg + (r2 - tl * fg);
  return out.t < T && out.n < n_tiles;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// MN-major fp32 operand: tf32 takes only the 128-byte swizzle with 32-byte atoms
// (SWIZZLE_128B_BASE32B, layout type 1; the TMA side is CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B):
// 512-byte atoms of 4 K rows x 32 frames.  A gathered group is 4 lags, stored as its 4
// frame blocks one atom after the other (LBO = 512 B along N); a K = 8 step takes two
// consecutive groups (SBO = one group's 2 KB along K).
__device__ __forceinline__ uint64_t desc_mn128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)(512 >> 4) << 16;             // LBO: next 32 frames
  d |= (uint64_t)((128 * GG * 4) >> 4) << 32;  // SBO: next 4 lags (the next group)
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;                      // SWIZZLE_128B_BASE32B
  return d;
}

// chunks of a tile with nk 64-lag blocks
// tile_nst[t] = the tile's 16-lag stages (its window K rounded up to 16, not to the 64-lag slab block)
__device__ __forceinline__ int num_chunks(int nst, int ch) { return (nst + ch - 1) / ch; }

__global__ void __launch_bounds__(kThreads, 1)
gather_tf32_kernel(const __grid_constant__ CUtensorMap ma_hi, const __grid_constant__ CUtensorMap ma_lo,
                   const __grid_constant__ CUtensorMap mb_hi, const __grid_constant__ CUtensorMap mb_lo, int b3d,
                   int fg, int CH, int u_begin, int u_end, int64_t F, int64_t J, int32_t T, const int32_t* __restrict__ group_col,
                   const int32_t* __restrict__ tile_blk, const int32_t* __restrict__ tile_nst,
                   const int32_t* __restrict__ tile_rows, float* __restrict__ zt, float* __restrict__ zg,
                   unsigned long long* __restrict__ keys) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)((F + GN - 1) / GN);
  const int u_total = min(u_end, ((n_tiles + fg - 1) / fg) * T * fg);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ma_hi);
    prefetch_tmap(&ma_lo);
    prefetch_tmap(&mb_hi);
    prefetch_tmap(&mb_lo);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.tfull[b], 1);
      mbar_init(&sm.tempty[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // lanes 0-7: one (plane, group) of gathered samples each; lanes 8-11: one (half, plane) slab
    constexpr uint32_t kBytes = 2u * (2 * GM * GK + GN * GK) * sizeof(float);
    const int plane = (lane >> 2) & 1, grp = lane & 3;
    const int ah = ((lane - 8) >> 1) & 1, ap = (lane - 8) & 1;
    // L2 policy: the unit group's gathered samples are re-read by every tile (keep them);
    // a tile's slabs only by the few CTAs on its frame tiles at about the same time
    const uint64_t keep = policy_evict_last(), once = policy_evict_first();
    auto next_unit = [&](int u, Unit& w) {
      while (u < u_total && !decode32(u, T, fg, n_tiles, w)) u += gridDim.x;
      return u;
    };
    auto stage_rows = [&](int buf, const Unit& w) {
      const int b0 = __ldg(tile_blk + w.t), nst = __ldg(tile_nst + w.t);
      for (int i = lane; i < nst * NG; i += 32) sm.rows[buf][i] = __ldg(group_col + b0 * (GB / GG) + i);
    };
    uint32_t g = 0;
    int buf = 0;
    Unit w;
    int u = next_unit(u_begin + blockIdx.x, w);
    if (u < u_total) stage_rows(0, w);
    while (u < u_total) {
      Unit wn;
      const int un = next_unit(u + gridDim.x, wn);
      if (un < u_total) stage_rows(buf ^ 1, wn);
      __syncwarp();
      const int b0 = __ldg(tile_blk + w.t), nst = __ldg(tile_nst + w.t);
      for (int kq = 0; kq < nst; ++kq, ++g) {     // 16-lag stages: a quarter block each
        const int blk = b0 + kq / (GB / GK), sub = kq % (GB / GK);
        const int row = sm.rows[buf][kq * NG + grp];
        const int s = g % NS;
        if (lane == 0) {
          mbar_wait(&sm.empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&sm.full[s], kBytes);
        }
        __syncwarp();
        if (lane < 8) {
          const CUtensorMap* mb = plane ? &mb_lo : &mb_hi;
          if (b3d) {
            tma_load_3d(sm.b[s][plane][grp], mb, &sm.full[s], 0, row, w.n * NA, keep);
          } else {
#pragma unroll
            for (int a = 0; a < NA; ++a)
              tma_load_2d(sm.b[s][plane][grp] + a * GA * GG, mb, &sm.full[s], w.n * GN + a * GA, row);
          }
        } else if (lane < 12) {
          tma_load_2d_hint(sm.a[s][ah][ap], ap ? &ma_lo : &ma_hi, &sm.full[s], sub * GK, (2 * blk + ah) * GM, once);
        }
      }
      __syncwarp();
      buf ^= 1;
      u = un;
      w = wn;
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // D f32, A/B tf32, A K-major, B MN-major (bit 16), N = 128, M = 128
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(GN >> 3) << 17) |
                                 ((uint32_t)(GM >> 4) << 24);
      uint32_t g = 0, c = 0;     // stage and chunk counters (chunk c uses TMEM buffer c & 1)
      for (int u = u_begin + blockIdx.x; u < u_total; u += gridDim.x) {
        Unit w;
        if (!decode32(u, T, fg, n_tiles, w)) continue;
        const int ns = __ldg(tile_nst + w.t);
        for (int kq = 0; kq < ns; ++kq, ++g) {
          const int s = g % NS;
          const int first = kq % CH == 0;
          if (first) {
            mbar_wait(&sm.tempty[c & 1], ((c >> 1) & 1) ^ 1);    // the epilogue folded this buffer
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          mbar_wait(&sm.full[s], (g / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dbuf = tmem + (c & 1) * 256;
#pragma unroll
          for (int k = 0; k < GK / UK; ++k) {
            const uint64_t aoff = (uint64_t)((k * UK * 4) >> 4);
            const uint64_t bh = desc_mn128(sm.b[s][0][2 * k]), bl = desc_mn128(sm.b[s][1][2 * k]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t d = dbuf + h * GN;
              const uint64_t a_h = smem_desc_sw64(sm.a[s][h][0]) + aoff, a_l = smem_desc_sw64(sm.a[s][h][1]) + aoff;
              mma_tf32(d, a_h, bh, idesc, (first && k == 0) ? 0u : 1u);
              mma_tf32(d, a_h, bl, idesc, 1u);
              mma_tf32(d, a_l, bh, idesc, 1u);
            }
          }
          mma_commit(&sm.empty[s]);
          if (kq % CH == CH - 1 || kq == ns - 1) {
            mma_commit(&sm.tfull[c & 1]);
            ++c;
          }
        }
      }
    }
  } else {
    // epilogue: warp = (half, TMEM lane quarter); each thread folds its candidate row's
    // 128 frames of every chunk into fp32 registers, then stores the unit's map (tile
    // order) and folds the per-frame argmax as the bf16 kernel's epilogue does
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * GN);
    const int64_t ldt = (int64_t)T * GT;
    uint32_t c = 0;
    for (int u = u_begin + blockIdx.x; u < u_total; u += gridDim.x) {
      Unit w;
      if (!decode32(u, T, fg, n_tiles, w)) continue;
      const int r = half * GM + q * 32 + lane;
      const int jrow = __ldg(tile_rows + (int64_t)w.t * GT + r);
      const int nc = num_chunks(__ldg(tile_nst + w.t), CH);
      float rs[GN];
      for (int j = 0; j < nc; ++j, ++c) {
        mbar_wait(&sm.tfull[c & 1], (c >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = lane_base + (c & 1) * 256;
#pragma unroll
        for (int cc = 0; cc < GN / 32; ++cc) {
          uint32_t rr[32];
          tmem_ld32(base + cc * 32, rr);
          if (j == 0) {
#pragma unroll
            for (int t = 0; t < 32; ++t) rs[cc * 32 + t] = __uint_as_float(rr[t]);
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) rs[cc * 32 + t] += __uint_as_float(rr[t]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[c & 1]);
      }
      const bool any = __any_sync(0xffffffffu, jrow >= 0);
      if (!any) continue;
#pragma unroll
      for (int cc = 0; cc < GN / 32; ++cc) {
        const int64_t f0 = (int64_t)w.n * GN + cc * 32;
        if (f0 >= F) break;
        if (zg) {
          if (jrow >= 0) {
            float* zc = zg + f0 * J + jrow;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (f0 + t < F) __stcs(zc + t * J, rs[cc * 32 + t]);
          }
        } else if (zt) {
          float* zc = zt + f0 * ldt + (int64_t)w.t * GT + r;
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (f0 + t < F) __stcs(zc + t * ldt, rs[cc * 32 + t]);
        }
        if (keys) {   // per frame: warp max of the ordered bits (redux), lowest winning lane (ballot)
          uint32_t best = 0u, win = 0u;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const uint32_t mine = jrow >= 0 ? ordered_bits(rs[cc * 32 + t]) : 0u;
            const uint32_t m = __reduce_max_sync(0xffffffffu, mine);
            const uint32_t who = __ballot_sync(0xffffffffu, mine == m);
            if (lane == t) {
              best = m;
              win = (uint32_t)(__ffs(who) - 1);
            }
          }
          const int jw = __shfl_sync(0xffffffffu, jrow, (int)win);
          if (f0 + lane < F && best != 0u)
            atomicMax(keys + f0 + lane,
                      ((unsigned long long)best << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)jw));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}
// ---- the same on CTA pairs (cta_group::2, a 2-CTA cluster per tile) ---------------------
// One tcgen05.mma.cta_group::2 (M = 256 candidates, N = 256 frames) covers the whole
// tile: CTA r of the pair holds tile half r (rows 128r..128r+127) of the slabs and frames
// 128r..128r+127 of the unit's gathered samples, so each SM streams half the operand bytes
// of the one-CTA kernel per MMA (32 KB per stage), and its accumulator is its 128
// candidates x 256 frames, which leaves room for the two fold buffers.  The leader (rank
// 0) issues the MMAs; both CTAs' TMA loads complete on the leader's stage barrier, the MMA
// commits arrive on both CTAs' barriers, and both CTAs' epilogues release a fold buffer on
// the leader's barrier.
//
// Two operand formats share the kernel (same bytes per stage, same barriers, same epilogue):
//   PairTf32: fp32 planes hi = tf32_rne(x), lo = tf32_rne(x - hi); kind::tf32, K = 8 per MMA,
//             16-lag stages, 4-lag gathered groups (512-byte MN atoms of 4 lags x 32 frames);
//   PairF16:  fp16 planes hi = f16_rne(x), lo = f16_rne(x - hi) -- the same 11 + 11
//             significant bits as the TF32 split while |x| stays in fp16 range (PHAT samples
//             are bounded by 2(K-1); the slab weights are scaled by a power of two on the
//             host and the epilogue undoes it exactly) -- kind::f16, K = 16 per MMA at twice
//             the TF32 rate, 32-lag stages, 8-lag groups (1 KB MN atoms of 8 lags x 64 frames).
constexpr int PN = 256;              // frames per unit (pair)
constexpr int PNC = PN / 2;          // frames per CTA (B half)
constexpr int PNS = 5;               // operand stages (32 KB each)
constexpr int PEpi = kEpi;           // epilogue warps
constexpr int PThreads = kThreads;
constexpr int PCols = PN / (PEpi / 4);         // accumulator columns folded per epilogue thread
constexpr int PGroupBytes = 2048;    // one (plane, group) of a CTA's 128 frames
constexpr int PSlabBytes = 8192;     // one plane of a CTA's slab half per stage
constexpr int PNG = 4;               // groups per stage

struct PairTf32 {
  static constexpr int GK = 16, GG = 4, UK = 8, GA = 32, ES = 4;
  static constexpr uint32_t kFmt = 2;          // instruction descriptor operand format: tf32
  // MN-major tf32 operand, 128-byte swizzle on 32-byte atoms: 512-byte atoms of 4 lags x 32 frames; a
  // group's four frame blocks follow one another (LBO = 512 B), the next 4 lags are the next
  // group, one (group, plane) pair further (SBO = 4 KB)
  static __device__ __forceinline__ uint64_t desc_b(const void* p) {
    const uint64_t addr = smem_u32(p);
    uint64_t d = 0;
    d |= (addr & 0x3FFFFull) >> 4;
    d |= (uint64_t)(512 >> 4) << 16;
    d |= (uint64_t)((2 * PGroupBytes) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;                    // SWIZZLE_128B_BASE32B
    return d;
  }
  static __device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
};

struct PairF16 {
  static constexpr int GK = 32, GG = 8, UK = 16, GA = 64, ES = 2;
  static constexpr uint32_t kFmt = 0;          // f16
  // MN-major fp16 operand, 128-byte swizzle: 1 KB atoms of 8 lags x 64 frames; a group's two
  // frame blocks follow one another (LBO = 1 KB along MN), the next 8 lags are the next group,
  // one (group, plane) pair further (SBO = 4 KB along K)
  static __device__ __forceinline__ uint64_t desc_b(const void* p) {
    const uint64_t addr = smem_u32(p);
    uint64_t d = 0;
    d |= (addr & 0x3FFFFull) >> 4;
    d |= (uint64_t)(1024 >> 4) << 16;
    d |= (uint64_t)((2 * PGroupBytes) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
    return d;
  }
  static __device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
};

template <class TR>
struct __align__(1024) PairSmem {
  unsigned char b[PNS][PNG][2][PGroupBytes];   // [group][plane] the CTA's frame blocks of one lag group (one TMA box per group)
  unsigned char a[PNS][2][PSlabBytes];         // [plane] this CTA's slab half (64-byte rows, 64-byte swizzle; one TMA box)
  float zs[PEpi][32 * 32];                     // [epilogue warp] 32 frames x 32 candidates of the map (128-byte swizzle) for a TMA store
  alignas(16) int32_t rows[2][kMaxBlocks * (GB / TR::GG)];   // the current / next unit's group rows
  uint64_t full[PNS], empty[PNS], tfull[2], tempty[2];
  uint32_t tmem_base;
};

template <class TR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PThreads, 1)
gather_pair_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                   const __grid_constant__ CUtensorMap mz, int z_tma, int l2pol, int64_t zt_ld, float zscale,
                   int fg, int tc, int CH, int u_begin, int u_end, int64_t F, int64_t J, int32_t T, const int32_t* __restrict__ group_col,
                   const int32_t* __restrict__ tile_blk, const int32_t* __restrict__ tile_nst,
                   const int32_t* __restrict__ tile_rows, float* __restrict__ zt, float* __restrict__ zg,
                   unsigned long long* __restrict__ keys) {
  constexpr int GK = TR::GK, GG = TR::GG, UK = TR::UK, GA = TR::GA, ES = TR::ES;
  constexpr int PNA = PNC / GA;                // frame blocks per group per CTA
  static_assert(GK / GG == PNG && PNC * GG * ES == PGroupBytes && GM * GK * ES == PSlabBytes, "stage geometry");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PairSmem<TR>& sm = *reinterpret_cast<PairSmem<TR>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int n_tiles = (int)((F + PN - 1) / PN);
  const int u_total = min(u_end, ((n_tiles + fg - 1) / fg) * fg * (tc > 0 ? ((T + tc - 1) / tc) * tc : T));

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ma);
    prefetch_tmap(&mb);
    for (int s = 0; s < PNS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.tfull[b], 1);
      mbar_init(&sm.tempty[b], 2 * PEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // The producer runs converged; per stage one elected lane issues this CTA's five TMA
    // loads -- four gathered lag groups (hi and lo planes in one 4D box each) and the slab
    // half (both planes in one 3D box) -- with operands on the uniform datapath.  (Ten
    // per-lane loads cost ~100 cycles each in ELECT / R2UR.BROADCAST loops and the producer,
    // not the tensor pipe, set the pace: ncu r2e.)
    constexpr uint32_t kBytes = 2u * (PSlabBytes + PNG * PGroupBytes);   // one CTA's stage
    // L2 policies (l2pol: diagnostic override, 2 bits each for the samples / slabs:
    // 0 evict_last, 1 evict_first, 2 evict_normal)
    auto pol = [](int c) { return c == 0 ? policy_evict_last() : c == 1 ? policy_evict_first() : policy_evict_normal(); };
    const uint64_t keep = pol(l2pol & 3), once = pol((l2pol >> 2) & 3);
    auto next_unit = [&](int u, Unit& w) {
      while (u < u_total && !decode_pair(u, T, fg, n_tiles, tc, w)) u += ncl;
      return u;
    };
    auto stage_rows = [&](int buf, const Unit& w) {
      const int b0 = __ldg(tile_blk + w.t), nst = __ldg(tile_nst + w.t);
      for (int i = lane; i < nst * PNG; i += 32) sm.rows[buf][i] = __ldg(group_col + b0 * (GB / GG) + i);
    };
    const uint32_t full0 = mapa_shared(smem_u32(&sm.full[0]), rank & ~1u);   // the leader's stage barriers
    uint32_t s = 0, ph = 1;
    int buf = 0;
    Unit w;
    int u = next_unit(u_begin + cid, w);
    if (u < u_total) stage_rows(0, w);
    while (u < u_total) {
      Unit wn;
      const int un = next_unit(u + ncl, wn);
      if (un < u_total) stage_rows(buf ^ 1, wn);
      __syncwarp();
      const int b0 = __ldg(tile_blk + w.t), nst = __ldg(tile_nst + w.t);
      const int fblk = w.n * (PN / GA) + (int)rank * PNA;
      for (int kq = 0; kq < nst; ++kq) {
        const int4 rows = *reinterpret_cast<const int4*>(&sm.rows[buf][kq * PNG]);
        mbar_wait(&sm.empty[s], ph);
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(&sm.full[s], 2 * kBytes);     // both CTAs' loads
          const uint32_t bar = full0 + s * (uint32_t)sizeof(uint64_t);
          tma_load_4d_pair(sm.b[s][0][0], &mb, bar, 0, rows.x, fblk, 0, keep);
          tma_load_4d_pair(sm.b[s][1][0], &mb, bar, 0, rows.y, fblk, 0, keep);
          tma_load_4d_pair(sm.b[s][2][0], &mb, bar, 0, rows.z, fblk, 0, keep);
          tma_load_4d_pair(sm.b[s][3][0], &mb, bar, 0, rows.w, fblk, 0, keep);
          tma_load_3d_pair(sm.a[s][0], &ma, bar, (kq % (GB / GK)) * GK, (2 * (b0 + kq / (GB / GK)) + (int)rank) * GM, 0, once);
        }
        __syncwarp();
        if (++s == PNS) {
          s = 0;
          ph ^= 1;
        }
      }
      __syncwarp();
      buf ^= 1;
      u = un;
      w = wn;
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // The pair's MMA issuer.  The whole warp runs the loop converged and one elected lane
      // issues (elect.sync keeps the descriptors on the uniform datapath; a lane-0 branch made
      // every tcgen05.mma an ELECT / R2UR.BROADCAST loop and the issuer, not the tensor pipe,
      // set the pace: ncu r2e).  Stage and chunk positions are running counters, and the
      // stage-0 descriptors are advanced by the stage pitch (address field = bytes >> 4).
      // D f32 [M = 256 frames (the pair)][N = 256 candidates]: A = the gathered samples, MN-major
      // (bit 15), B = the slabs, K-major -- an accumulator lane is a frame, so the epilogue's
      // argmax runs down a thread's registers and a thread's candidates are contiguous map bytes
      constexpr uint32_t idesc = (1u << 4) | (TR::kFmt << 7) | (TR::kFmt << 10) | (1u << 15) |
                                 ((uint32_t)((2 * GM) >> 3) << 17) | ((uint32_t)(PN >> 4) << 24);
      constexpr int NK = GK / UK;
      constexpr uint64_t kAPitch = sizeof(sm.a[0]) >> 4, kBPitch = sizeof(sm.b[0]) >> 4;
      const uint64_t a0h = smem_desc_sw64(sm.a[0][0]), a0l = smem_desc_sw64(sm.a[0][1]);
      uint64_t b0h[NK], b0l[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        b0h[k] = TR::desc_b(sm.b[0][2 * k][0]);
        b0l[k] = TR::desc_b(sm.b[0][2 * k][1]);
      }
      uint32_t s = 0, ph = 0, c = 0;
      for (int u = u_begin + cid; u < u_total; u += ncl) {
        Unit w;
        if (!decode_pair(u, T, fg, n_tiles, tc, w)) continue;
        const int ns = __ldg(tile_nst + w.t);
        int kc = 0;                                              // stage within the accumulation chunk
        for (int kq = 0; kq < ns; ++kq) {
          if (kc == 0) {
            mbar_wait(&sm.tempty[c & 1], ((c >> 1) & 1) ^ 1);    // both epilogues folded this buffer
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          mbar_wait(&sm.full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const bool last = kc == CH - 1 || kq == ns - 1;
          if (elect_one()) {
            const uint32_t d = tmem + (c & 1) * PN;
            const uint64_t ao = (uint64_t)s * kAPitch, bo = (uint64_t)s * kBPitch;
#pragma unroll
            for (int k = 0; k < NK; ++k) {
              const uint64_t aoff = ao + (uint64_t)((k * UK * ES) >> 4);
              TR::mma(d, b0h[k] + bo, a0h + aoff, idesc, (kc == 0 && k == 0) ? 0u : 1u);
              TR::mma(d, b0l[k] + bo, a0h + aoff, idesc, 1u);
              TR::mma(d, b0h[k] + bo, a0l + aoff, idesc, 1u);
            }
            mma_commit_pair(&sm.empty[s]);
            if (last) mma_commit_pair(&sm.tfull[c & 1]);
          }
          __syncwarp();
          if (last) {
            ++c;
            kc = 0;
          } else {
            ++kc;
          }
          if (++s == PNS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else {
    // epilogue: warp = (column half ch, TMEM lane quarter q): this CTA's frames 32q..32q+31, one
    // per lane, x tile rows 128ch..128ch+127 in the thread's registers.  Every chunk is folded
    // into fp32 registers; then the argmax runs down the registers (no cross-lane work), and
    // the map leaves in 32-candidate slices through the warp's own swizzled staging tile and a
    // TMA store (tile order), or as whole 32-byte runs (grid order).
    const int q = warp & 3;
    const int ch = (warp - 2) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ch * PCols);
    // map stores stream past L2 (evict_first): they must not push out the group's samples
    const uint64_t zpol = ((l2pol >> 4) & 3) == 0 ? policy_evict_first()
                          : ((l2pol >> 4) & 3) == 1 ? policy_evict_normal() : policy_evict_last();
    float* zsw = sm.zs[warp - 2];
    uint32_t c = 0;
    for (int u = u_begin + cid; u < u_total; u += ncl) {
      Unit w;
      if (!decode_pair(u, T, fg, n_tiles, tc, w)) continue;
      const int64_t f0 = (int64_t)w.n * PN + (int)rank * PNC + q * 32;   // the warp's first frame
      const int64_t f = f0 + lane;
      const int32_t* trow = tile_rows + (int64_t)w.t * GT + ch * PCols;
      // the tile's valid rows are a prefix: count this column half's
      int nv = 0;
#pragma unroll
      for (int i = 0; i < PCols / 32; ++i) nv += __ldg(trow + i * 32 + lane) >= 0 ? 1 : 0;
      nv = __reduce_add_sync(0xffffffffu, nv);
      const int nc = num_chunks(__ldg(tile_nst + w.t), CH);
      float rs[PCols];
      for (int j = 0; j < nc; ++j, ++c) {
        mbar_wait(&sm.tfull[c & 1], (c >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = lane_base + (c & 1) * PN;
#pragma unroll
        for (int cc = 0; cc < PCols / 32; ++cc) {
          uint32_t rr[32];
          tmem_ld32(base + cc * 32, rr);
          if (j == 0) {
#pragma unroll
            for (int t = 0; t < 32; ++t) rs[cc * 32 + t] = __uint_as_float(rr[t]);
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) rs[cc * 32 + t] += __uint_as_float(rr[t]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&sm.tempty[c & 1]), rank & ~1u));
      }
      if (nv == 0 || f0 >= F) continue;                // padding rows only / frames past the batch
      if (zscale != 1.0f) {   // undo the slabs' power-of-two scale (exact)
#pragma unroll
        for (int t = 0; t < PCols; ++t) rs[t] *= zscale;
      }
      if (keys) {   // first maximum of the thread's valid candidates (rows ascend with the candidate)
        float bv = rs[0];
        int bc = 0;
        if (nv == PCols) {
#pragma unroll
          for (int t = 1; t < PCols; ++t)
            if (rs[t] > bv) {
              bv = rs[t];
              bc = t;
            }
        } else {
#pragma unroll
          for (int t = 1; t < PCols; ++t)
            if (t < nv && rs[t] > bv) {
              bv = rs[t];
              bc = t;
            }
        }
        if (f < F) atomicMax(keys + f, make_key(bv, (uint32_t)__ldg(trow + bc)));
      }
      if (z_tma) {
#pragma unroll
        for (int cc = 0; cc < PCols / 32; ++cc) {
          if (cc * 32 >= nv) break;                    // uniform over the warp
          if (lane == 0) bulk_wait_read<0>();          // the previous slice has left the staging tile
          __syncwarp();
          // row = this lane's frame (128 B); 16-byte chunk j sits at j ^ (row & 7) (SWIZZLE_128B)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(zsw + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                make_float4(rs[cc * 32 + 4 * j], rs[cc * 32 + 4 * j + 1], rs[cc * 32 + 4 * j + 2],
                            rs[cc * 32 + 4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (z_tma == 2)   // contiguous tiles: straight into the grid-order map (rows / columns clipped)
              tma_store_2d_hint(&mz, zsw, w.t * GT + ch * PCols + cc * 32, (int)f0, zpol);
            else
              tma_store_4d_hint(&mz, zsw, ch * PCols + cc * 32, 0, w.t,
                                w.n * (PN / 32) + (int)rank * (PNC / 32) + q, zpol);
            bulk_commit();
          }
        }
      } else if (zg) {   // grid order: the tile's rows are aligned runs of 8 candidates
        if (f < F) {
          float* zf = zg + f * J;
#pragma unroll
          for (int r8 = 0; r8 < PCols / 8; ++r8) {
            const int j8 = __ldg(trow + r8 * 8);
            if (j8 >= 0) {
              st_global_v4_hint(zf + j8, rs[r8 * 8], rs[r8 * 8 + 1], rs[r8 * 8 + 2], rs[r8 * 8 + 3], zpol);
              st_global_v4_hint(zf + j8 + 4, rs[r8 * 8 + 4], rs[r8 * 8 + 5], rs[r8 * 8 + 6], rs[r8 * 8 + 7], zpol);
            }
          }
        }
      } else if (zt) {   // tile order by register stores (diagnostic: SRPGPU_GATHER_ZSTG)
        if (f < F) {
          // zt_ld == 0: diagnostic, every unit to one block
          const int64_t blk = zt_ld == 0 ? 0 : (int64_t)(w.n * (PN / 32) + (int)rank * (PNC / 32) + q) * T + w.t;
          float* zc = zt + (blk * 32 + lane) * GT + ch * PCols;
#pragma unroll
          for (int t = 0; t < PCols; t += 4)
            st_global_v4_hint(zc + t, rs[t], rs[t + 1], rs[t + 2], rs[t + 3], zpol);
        }
      }
    }
    if (lane == 0) bulk_wait_all();                    // the map's TMA stores have landed
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}
}  // namespace g32

#ifndef UNTILE_U
#define UNTILE_U 4
#endif

// tile order -> grid order: z[f][j] = zt[f][pos[j]] (coalesced writes; the reads follow
// the tiles' ascending rows, mostly short contiguous runs).  FB frames per CTA share each
// thread's pos loads (the kernel is L1-wavefront bound: ncu r1j, L1 86% of peak)
// blocked != 0 (the pair kernel): the tile-order map is stored in blocks of ZB = 32 frames,
// zt[frame block][tile][32 frames][256 rows], so an epilogue warp's 32 frames x 128 candidates
// land in one 32 KB block (with the frames' rows 1.3 MB apart the stores' latency stalled the
// pair kernel's accumulator hand-back: +4.5 ms at cfg4; whole 256-frame units, on the other
// hand, scatter this pass's reads over 343 MB per frame: 6.3 -> 14.4 ms); blocked = the number
// of tiles T.
constexpr int ZB = 32;
template <int FB>
__global__ void __launch_bounds__(256) untile_kernel(const float* __restrict__ zt, int64_t ldt, const int32_t* __restrict__ pos, int64_t J,
                              int64_t F, float* __restrict__ z, int64_t blocked) {
  constexpr int U = UNTILE_U;   // independent gathers in flight per thread (per frame)
  for (int64_t f0 = (int64_t)blockIdx.y * FB; f0 < F; f0 += (int64_t)gridDim.y * FB) {
    const int nf = F - f0 < FB ? (int)(F - f0) : FB;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < J; j0 += U * step) {
      int64_t p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t q = j0 + u * step < J ? __ldg(pos + j0 + u * step) : 0;
        p[u] = blocked ? (int64_t)(q >> 8) * (GT * ZB) + (q & 255) : (int64_t)q;
      }
#pragma unroll
      for (int fb = 0; fb < FB; ++fb) {
        if (fb < nf) {
          const int64_t f = f0 + fb;
          const float* src = blocked ? zt + ((f / ZB) * blocked * ZB + (f % ZB)) * GT : zt + f * ldt;
          float* dst = z + (f0 + fb) * J;
          float v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = __ldcs(src + p[u]);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + u * step < J) __stcs(dst + j0 + u * step, v[u]);
        }
      }
    }
  }
}

// frames per CTA of the untile pass (tuning override: SRPGPU_UNTILE_FB=1|2|4).  4 frames share
// each pos load on large batches (cfg4, 10^4 frames: map + untile 33.8 -> 33.4 ms); small
// batches keep 1 (the cfg5 sweep at 16-256 frames lost 7-11% with 4: fewer CTAs per frame)
static int untile_frames(int64_t num_frames) {
  static const int forced = [] {
    const char* v = std::getenv("SRPGPU_UNTILE_FB");
    const int x = v ? std::atoi(v) : 0;
    return (x == 1 || x == 2 || x == 4 || x == 8) ? x : 0;
  }();
  if (forced) return forced;
  return num_frames >= 4096 ? 4 : 1;
}

static int untile(const float* z_tiles, int32_t num_tiles, const int32_t* tile_pos, int64_t num_candidates,
                  int64_t num_frames, float* z, cudaStream_t st, bool blocked = false) {
  const int fb = untile_frames(num_frames);
  dim3 grid((unsigned)std::min<int64_t>((num_candidates + 255) / 256, 64),
            (unsigned)std::min<int64_t>((num_frames + fb - 1) / fb, 65535));
  const int64_t ldt = (int64_t)num_tiles * GT;
  const int64_t bt = blocked ? num_tiles : 0;
  if (fb == 8) untile_kernel<8><<<grid, 256, 0, st>>>(z_tiles, ldt, tile_pos, num_candidates, num_frames, z, bt);
  else if (fb == 4) untile_kernel<4><<<grid, 256, 0, st>>>(z_tiles, ldt, tile_pos, num_candidates, num_frames, z, bt);
  else if (fb == 2) untile_kernel<2><<<grid, 256, 0, st>>>(z_tiles, ldt, tile_pos, num_candidates, num_frames, z, bt);
  else untile_kernel<1><<<grid, 256, 0, st>>>(z_tiles, ldt, tile_pos, num_candidates, num_frames, z, bt);
  SRPGPU_CHECK_LAUNCH("interp_map_gather(untile)");
  return SRPGPU_OK;
}

}  // namespace gtc

int reset_keys(uint64_t* keys, int64_t F, cudaStream_t st);

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_interp_map_gather_tc(const void* samples_planes, int64_t num_frames, int32_t num_cols,
                                           int64_t planes_ld,
                                           const void* slab_planes, int64_t num_slabs, const int32_t* group_col,
                                           const int32_t* tile_slab, const int32_t* tile_nkb,
                                           const int32_t* tile_rows, int32_t num_tiles, int64_t num_candidates,
                                           int32_t num_ctas, const int32_t* tile_pos,
                                           float* z_tiles, float* z, uint64_t* keys, srpgpu_stream_t stream) {
  using namespace gtc;
  SRPGPU_CHECK_ARG(num_frames >= 0 && num_cols >= 1 && planes_ld >= num_frames && planes_ld % 8 == 0 &&
                       num_slabs >= 0 && num_tiles >= 0 && num_candidates >= 1 && num_ctas >= 0,
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_tc: bad shape");
  SRPGPU_CHECK_ARG(((uintptr_t)samples_planes & 15) == 0 && ((uintptr_t)slab_planes & 15) == 0 &&
                       ((uintptr_t)group_col & 15) == 0,
                   SRPGPU_ERR_VALUE, "interp_map_gather_tc: operands must be 16-byte aligned");
  SRPGPU_CHECK_ARG(num_frames < (1ll << 31) && num_candidates < (1ll << 31) && num_slabs * GM < (1ll << 31),
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_tc: too large");
  SRPGPU_CHECK_ARG(!z || !z_tiles || tile_pos, SRPGPU_ERR_VALUE,
                   "interp_map_gather_tc: a tile-order map needs tile_pos");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames == 0 || num_tiles == 0 || num_ctas == 0) return SRPGPU_OK;
  const auto* xs = reinterpret_cast<const uint16_t*>(samples_planes);
  const auto* xo = reinterpret_cast<const uint16_t*>(slab_planes);
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int64_t arows = num_slabs * GM;
  const CUtensorMapSwizzle sw64 = CU_TENSOR_MAP_SWIZZLE_64B;
  if ((s = make_map_2d(&ma_hi, bf, 2, xo, arows, GB, GB, GK, GM, "interp_map_gather_tc", sw64)) ||
      (s = make_map_2d(&ma_lo, bf, 2, xo + arows * GB, arows, GB, GB, GK, GM, "interp_map_gather_tc", sw64)) ||
      (s = make_map_2d(&mb_hi, bf, 2, xs, num_cols, num_frames, planes_ld, GA, GG, "interp_map_gather_tc")) ||
      (s = make_map_2d(&mb_lo, bf, 2, xs + (int64_t)((num_cols + 7) / 8 * 8) * planes_ld, num_cols, num_frames,
                       planes_ld, GA, GG, "interp_map_gather_tc")))   // planes hold round8(S) rows each
    return s;
  const size_t smem = sizeof(Smem) + 1024;
  if (cudaFuncSetAttribute(gather_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("interp_map_gather_tc: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  gather_tc_kernel<<<(unsigned)num_ctas, kThreads, smem, st>>>(
      ma_hi, ma_lo, mb_hi, mb_lo, num_frames, num_candidates, num_tiles, group_col, tile_slab, tile_nkb, tile_rows,
      z ? z_tiles : nullptr, z && !z_tiles ? z : nullptr, reinterpret_cast<unsigned long long*>(keys));
  SRPGPU_CHECK_LAUNCH("interp_map_gather_tc");
  if (z && z_tiles && (s = gtc::untile(z_tiles, num_tiles, tile_pos, num_candidates, num_frames, z, st))) return s;
  return SRPGPU_OK;
}

namespace srpgpu {
namespace gtc {

// tuning overrides shared by the gathered-window entry points
struct GatherTuning {
  int pair;                   // CTA pairs (SRPGPU_GATHER_PAIR=0: the one-CTA kernel)
  int64_t frames_per_group;   // frames whose gathered samples stay L2-resident (SRPGPU_GATHER_GROUP)
  int chunk;                  // stages per TMEM accumulation chunk (SRPGPU_GATHER_CHUNK)
  int l2pol;                  // L2 policies (SRPGPU_GATHER_L2)
  int64_t zt_ld;              // diagnostic: SRPGPU_GATHER_ZTEST=1 writes every frame's row to the same place
  int zstg;                   // SRPGPU_GATHER_ZSTG: tile-order map by register stores instead of TMA stores
  int tchunk;                 // tiles per L2-resident slab chunk (SRPGPU_GATHER_TCHUNK; 0: frame-group-major units)
};

static const GatherTuning& tuning() {
  static const GatherTuning t = [] {
    GatherTuning g;
    const char* v = getenv("SRPGPU_GATHER_PAIR");
    g.pair = v ? atoi(v) : 1;
    v = getenv("SRPGPU_GATHER_GROUP");
    const int64_t x = v ? atoll(v) : 0;
    // 0: per operand format (launch_pair): the group's hi / lo samples (F_g x S x 4 B in fp16, 8 B in
    // fp32) stay L2-resident next to the slabs in flight
    g.frames_per_group = x >= 256 && x % 256 == 0 ? x : (int64_t)0;
    v = getenv("SRPGPU_GATHER_CHUNK");
    const int c = v ? atoi(v) : 0;
    g.chunk = c >= 1 && c <= 64 ? c : 8;
    // samples evict_last, slabs evict_first, map stores evict_first (bits 0-1 / 2-3 / 4-5).  cfg4,
    // fp16x3, 10^4 frames (profiles/r2h_gather_f16_traffic*.log, DRAM reads / kernel time under
    // ncu): slabs evict_normal 58.5 GB / 16.2 ms, slabs evict_first 45.1 GB / 14.7 ms, and with
    // 512-frame groups 40.1 GB / 14.5 ms; map stores evict_normal: 57 GB / 15.2 ms
    g.l2pol = getenv("SRPGPU_GATHER_L2") ? atoi(getenv("SRPGPU_GATHER_L2")) : (0 | (1 << 2));
    g.zt_ld = getenv("SRPGPU_GATHER_ZTEST") ? 0 : -1;
    g.zstg = getenv("SRPGPU_GATHER_ZSTG") ? 1 : 0;
    g.tchunk = getenv("SRPGPU_GATHER_TCHUNK") ? atoi(getenv("SRPGPU_GATHER_TCHUNK")) : 0;
    return g;
  }();
  return t;
}

// co-resident 2-CTA clusters of the pair kernel (0: it cannot run here)
template <class TR>
static int pair_clusters(int num_ctas, cudaStream_t st) {
  const size_t psmem = sizeof(g32::PairSmem<TR>) + 1024;
  if (cudaFuncSetAttribute(g32::gather_pair_kernel<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(num_ctas & ~1));
  cfg.blockDim = dim3(g32::PThreads);
  cfg.dynamicSmemBytes = psmem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, g32::gather_pair_kernel<TR>, &cfg) != cudaSuccess) clusters = 0;
  cudaGetLastError();
  return std::min(clusters, num_ctas / 2);
}

// operand maps of the pair kernel, hi and lo planes in one box each: the slabs
// [2][num_slabs * 128][64] as {lags, rows, planes} (64-byte swizzle, one stage of GK lags of the
// CTA's 128 rows per box) and the lag-major sample planes [2][round8(S)][planes_ld] as {GA
// frames, lags, frame blocks, planes} (one box per gathered group: the CTA's frame blocks of
// GG lag rows, both planes)
template <class TR>
static int pair_maps(CUtensorMapDataType dt, const void* samples_planes, int32_t num_cols, int64_t planes_ld,
                     const void* slab_planes, int64_t num_slabs, CUtensorMap* ma, CUtensorMap* mb, const char* what) {
  const int64_t arows = num_slabs * GM;
  const int64_t c8 = (int64_t)((num_cols + 7) / 8 * 8);   // planes hold round8(S) rows each
  int s;
  {
    const int64_t dims[3] = {GB, arows, 2};
    const int box[3] = {TR::GK, GM, 2};
    if ((s = make_map_3d(ma, dt, slab_planes, dims, (int64_t)GB * TR::ES, arows * GB * TR::ES, box, what,
                         CU_TENSOR_MAP_SWIZZLE_64B)))
      return s;
  }
  const CUtensorMapSwizzle swz = TR::ES == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  const int64_t dims[4] = {TR::GA, num_cols, planes_ld / TR::GA, 2};
  const int64_t strides[3] = {planes_ld * TR::ES, (int64_t)TR::GA * TR::ES, c8 * planes_ld * TR::ES};
  const int box[4] = {TR::GA, TR::GG, g32::PNC / TR::GA, 2};
  return make_map_4d(mb, dt, samples_planes, dims, strides, box, what, swz);
}

template <class TR>
static int launch_pair(int clusters, const CUtensorMap& ma, const CUtensorMap& mb, float zscale, int64_t num_frames, int64_t num_candidates,
                       int32_t num_tiles, const int32_t* group_col, const int32_t* tile_slab, const int32_t* tile_nst,
                       const int32_t* tile_rows, float* z_tiles, float* z, uint64_t* keys, cudaStream_t st,
                       const char* what, bool contiguous = false) {
  const GatherTuning& tn = tuning();
  // tile-order map through TMA stores in blocks of 32 frames ([frame block][tile][32 frames][256
  // rows]): box of 32 candidates x 32 frames (an epilogue warp's 128-byte-swizzled staging tile)
  CUtensorMap mz = ma;
  int z_tma = 0, s;
  if (z_tiles && !tn.zstg) {
    const int64_t dims[4] = {GT, ZB, num_tiles, (num_frames + ZB - 1) / ZB};
    const int64_t strides[3] = {(int64_t)GT * 4, (int64_t)GT * ZB * 4, (int64_t)GT * ZB * 4 * num_tiles};
    const int box[4] = {32, 32, 1, 1};
    if ((s = make_map_4d(&mz, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z_tiles, dims, strides, box, what,
                         CU_TENSOR_MAP_SWIZZLE_128B)))
      return s;
    z_tma = 1;
  } else if (z && contiguous && num_candidates % 4 == 0) {
    // tiles of 256 consecutive candidates: the same staging tiles go straight into z [F][J]
    if ((s = make_map_2d(&mz, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, z, num_frames, num_candidates, num_candidates,
                         32, 32, what, CU_TENSOR_MAP_SWIZZLE_128B)))
      return s;
    z_tma = 2;
  }
  const int64_t fpg = tn.frames_per_group ? tn.frames_per_group : (TR::ES == 2 ? 512 : 1024);
  const int fg = (int)(fpg / g32::PN);
  const int tc = tn.tchunk > 0 ? tn.tchunk : 0;
  const int64_t tiles_padded = tc > 0 ? ((int64_t)num_tiles + tc - 1) / tc * tc : num_tiles;
  const int64_t units_per_group = tiles_padded * fg;
  const int64_t n_groups = (num_frames + fpg - 1) / fpg;
  SRPGPU_CHECK_ARG(n_groups * units_per_group < (1ll << 31), SRPGPU_ERR_DIMENSION, "%s: too many units", what);
  g32::gather_pair_kernel<TR><<<(unsigned)(2 * clusters), g32::PThreads, sizeof(g32::PairSmem<TR>) + 1024, st>>>(
      ma, mb, mz, tn.zt_ld < 0 ? z_tma : 0, tn.l2pol, tn.zt_ld, zscale, fg, tc, tn.chunk, 0,
      (int)(n_groups * units_per_group), num_frames, num_candidates, num_tiles, group_col, tile_slab, tile_nst,
      tile_rows, z_tiles, z && !z_tiles ? z : nullptr, reinterpret_cast<unsigned long long*>(keys));
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

}  // namespace gtc
}  // namespace srpgpu

extern "C" int srpgpu_interp_map_gather_tf32(const float* samples_planes, int64_t num_frames, int32_t num_cols,
                                             int64_t planes_ld, const float* slab_planes, int64_t num_slabs,
                                             const int32_t* group_col, const int32_t* tile_slab,
                                             const int32_t* tile_nkb, const int32_t* tile_rows, int32_t num_tiles,
                                             int64_t num_candidates, int32_t num_ctas, const int32_t* tile_pos,
                                             float* z_tiles, float* z, uint64_t* keys, srpgpu_stream_t stream) {
  using namespace gtc;
  SRPGPU_CHECK_ARG(num_frames >= 0 && num_cols >= 1 && planes_ld >= num_frames && planes_ld % 32 == 0 &&
                       num_slabs >= 0 && num_tiles >= 0 && num_candidates >= 1 && num_ctas >= 0,
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_tf32: bad shape (planes pitch: a multiple of 32 >= F)");
  SRPGPU_CHECK_ARG(((uintptr_t)samples_planes & 127) == 0 && ((uintptr_t)slab_planes & 15) == 0 &&
                       ((uintptr_t)group_col & 15) == 0,
                   SRPGPU_ERR_VALUE, "interp_map_gather_tf32: operands must be aligned (samples 128 B, slabs 16 B)");
  SRPGPU_CHECK_ARG(num_frames < (1ll << 31) && num_candidates < (1ll << 31) && num_slabs * GM < (1ll << 31),
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_tf32: too large");
  SRPGPU_CHECK_ARG(!z || !z_tiles || tile_pos, SRPGPU_ERR_VALUE,
                   "interp_map_gather_tf32: a tile-order map needs tile_pos");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames == 0 || num_tiles == 0 || num_ctas == 0) return SRPGPU_OK;
  const GatherTuning& tn = tuning();
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  const CUtensorMapDataType f32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  // CTA pairs (cta_group::2) unless SRPGPU_GATHER_PAIR=0, the 3D sample view cannot be encoded
  // or no 2-CTA cluster fits; persistent grid = the co-resident clusters
  int clusters = 0;
  if (tn.pair && !getenv("SRPGPU_GATHER_2D") &&
      pair_maps<g32::PairTf32>(f32, samples_planes, num_cols, planes_ld, slab_planes, num_slabs, &ma_hi, &mb_hi,
                               "interp_map_gather_tf32") == SRPGPU_OK)
    clusters = pair_clusters<g32::PairTf32>(num_ctas, st);
  if (clusters > 0) {
    if ((s = launch_pair<g32::PairTf32>(clusters, ma_hi, mb_hi, 1.0f, num_frames, num_candidates,
                                        num_tiles, group_col, tile_slab, tile_nkb, tile_rows, z_tiles, z, keys, st,
                                        "interp_map_gather_tf32", z && !z_tiles && !tile_pos)))
      return s;
  } else {
    // one-CTA fallback (N = 128 frames per unit)
    const int64_t arows = num_slabs * GM;
    const int64_t c8 = (int64_t)((num_cols + 7) / 8 * 8);
    const float* xs_lo = samples_planes + c8 * planes_ld;
    if ((s = make_map_2d(&ma_hi, f32, 4, slab_planes, arows, GB, GB, g32::GK, GM, "interp_map_gather_tf32",
                         CU_TENSOR_MAP_SWIZZLE_64B)) ||
        (s = make_map_2d(&ma_lo, f32, 4, slab_planes + arows * GB, arows, GB, GB, g32::GK, GM,
                         "interp_map_gather_tf32", CU_TENSOR_MAP_SWIZZLE_64B)))
      return s;
    const CUtensorMapSwizzle sw32 = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    int b3d = getenv("SRPGPU_GATHER_2D") ? 0 : 1;
    {
      const int64_t dims[3] = {g32::GA, num_cols, planes_ld / g32::GA};
      const int box[3] = {g32::GA, g32::GG, g32::NA};
      if (make_map_3d(&mb_hi, f32, samples_planes, dims, planes_ld * 4, g32::GA * 4, box, "interp_map_gather_tf32",
                      sw32) ||
          make_map_3d(&mb_lo, f32, xs_lo, dims, planes_ld * 4, g32::GA * 4, box, "interp_map_gather_tf32", sw32))
        b3d = 0;
    }
    if (!b3d && ((s = make_map_2d(&mb_hi, f32, 4, samples_planes, num_cols, num_frames, planes_ld, g32::GA, g32::GG,
                                  "interp_map_gather_tf32", sw32)) ||
                 (s = make_map_2d(&mb_lo, f32, 4, xs_lo, num_cols, num_frames, planes_ld, g32::GA, g32::GG,
                                  "interp_map_gather_tf32", sw32))))
      return s;
    const size_t smem = sizeof(g32::Smem) + 1024;
    if (cudaFuncSetAttribute(g32::gather_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("interp_map_gather_tf32: cannot reserve %zu B shared memory", smem);
      return SRPGPU_ERR_LAUNCH;
    }
    const int64_t fpg = tn.frames_per_group ? tn.frames_per_group : 1024;
    const int fg = (int)(fpg / g32::GN);
    const int64_t units_per_group = (int64_t)num_tiles * fg;
    const int64_t n_groups = (num_frames + fpg - 1) / fpg;
    SRPGPU_CHECK_ARG(n_groups * units_per_group < (1ll << 31), SRPGPU_ERR_DIMENSION,
                     "interp_map_gather_tf32: too many units");
    g32::gather_tf32_kernel<<<(unsigned)num_ctas, kThreads, smem, st>>>(
        ma_hi, ma_lo, mb_hi, mb_lo, b3d, fg, tn.chunk, 0, (int)(n_groups * units_per_group), num_frames,
        num_candidates, num_tiles, group_col, tile_slab, tile_nkb, tile_rows, z ? z_tiles : nullptr,
        z && !z_tiles ? z : nullptr, reinterpret_cast<unsigned long long*>(keys));
    SRPGPU_CHECK_LAUNCH("interp_map_gather_tf32");
  }
  // one launch over every group; the untile pass follows (measured: running group g's untile
  // on a side stream under group g + 1's gather launch was slower, 50 vs 42 ms at cfg4 --
  // the two contend for the SMs' issue slots and L2)
  if (z && z_tiles && (s = untile(z_tiles, num_tiles, tile_pos, num_candidates, num_frames, z, st, clusters > 0))) return s;
  return SRPGPU_OK;
}

// The same map in fp16x3 (PairF16): samples_planes fp16 [2][round8(S)][planes_ld] (hi / lo,
// lag-major, natural lag order, planes_ld a multiple of 64), slab_planes fp16
// [2][num_slabs * 128][64] = split of (slab * 1 / z_scale) with z_scale a power of two; the
// layout's groups are 8 lags and tile_nst counts 32-lag stages.  CTA pairs only.
extern "C" int srpgpu_interp_map_gather_f16(const void* samples_planes, int64_t num_frames, int32_t num_cols,
                                            int64_t planes_ld, const void* slab_planes, int64_t num_slabs,
                                            const int32_t* group_col, const int32_t* tile_slab,
                                            const int32_t* tile_nst, const int32_t* tile_rows, int32_t num_tiles,
                                            int64_t num_candidates, int32_t num_ctas, const int32_t* tile_pos,
                                            float z_scale, float* z_tiles, float* z, uint64_t* keys,
                                            srpgpu_stream_t stream) {
  using namespace gtc;
  SRPGPU_CHECK_ARG(num_frames >= 0 && num_cols >= 1 && planes_ld >= num_frames && planes_ld % 64 == 0 &&
                       num_slabs >= 0 && num_tiles >= 0 && num_candidates >= 1 && num_ctas >= 0,
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_f16: bad shape (planes pitch: a multiple of 64 >= F)");
  SRPGPU_CHECK_ARG(((uintptr_t)samples_planes & 127) == 0 && ((uintptr_t)slab_planes & 15) == 0 &&
                       ((uintptr_t)group_col & 15) == 0,
                   SRPGPU_ERR_VALUE, "interp_map_gather_f16: operands must be aligned (samples 128 B, slabs 16 B)");
  SRPGPU_CHECK_ARG(num_frames < (1ll << 31) && num_candidates < (1ll << 31) && num_slabs * GM < (1ll << 31),
                   SRPGPU_ERR_DIMENSION, "interp_map_gather_f16: too large");
  SRPGPU_CHECK_ARG(!z || !z_tiles || tile_pos, SRPGPU_ERR_VALUE, "interp_map_gather_f16: a tile-order map needs tile_pos");
  SRPGPU_CHECK_ARG(z_scale > 0.f, SRPGPU_ERR_VALUE, "interp_map_gather_f16: z_scale must be positive");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames == 0 || num_tiles == 0 || num_ctas == 0) return SRPGPU_OK;
  CUtensorMap ma, mb;
  if ((s = pair_maps<g32::PairF16>(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, samples_planes, num_cols, planes_ld, slab_planes,
                                   num_slabs, &ma, &mb, "interp_map_gather_f16")))
    return s;
  const int clusters = pair_clusters<g32::PairF16>(num_ctas, st);
  if (clusters == 0) {
    set_error("interp_map_gather_f16: no 2-CTA cluster of the pair kernel fits this device");
    return SRPGPU_ERR_LAUNCH;
  }
  if ((s = launch_pair<g32::PairF16>(clusters, ma, mb, z_scale, num_frames, num_candidates,
                                     num_tiles, group_col, tile_slab, tile_nst, tile_rows, z_tiles, z, keys, st,
                                     "interp_map_gather_f16", z && !z_tiles && !tile_pos)))
    return s;
  if (z && z_tiles && (s = untile(z_tiles, num_tiles, tile_pos, num_candidates, num_frames, z, st, true))) return s;
  return SRPGPU_OK;
}

// The gather pass alone: z[f][j] = z_tiles[f][tile_pos[j]], for a scratch map an earlier
// srpgpu_interp_map_gather_* call left (z NULL there, z_tiles given).  blocked != 0: the CTA-pair
// kernels' layout ([frame block of 32][tile][32 frames][256 rows]); 0: rows of num_tiles * 256.
extern "C" int srpgpu_interp_map_untile(const float* z_tiles, int32_t num_tiles, const int32_t* tile_pos,
                                        int64_t num_candidates, int64_t num_frames, float* z, int32_t blocked,
                                        srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_tiles >= 0 && num_candidates >= 0 && num_frames >= 0, SRPGPU_ERR_DIMENSION,
                   "interp_map_untile: bad shape");
  SRPGPU_CHECK_ARG(z_tiles && tile_pos && z, SRPGPU_ERR_VALUE, "interp_map_untile: null argument");
  if (num_frames == 0 || num_candidates == 0) return SRPGPU_OK;
  return srpgpu::gtc::untile(z_tiles, num_tiles, tile_pos, num_candidates, num_frames, z, as_stream(stream),
                             blocked != 0);
}
