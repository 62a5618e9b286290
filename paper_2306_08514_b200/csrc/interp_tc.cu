// Interpolation maps (si_map / sspi_map, interpolation.py:112-136, 188-195) on the
// 5th-generation tensor cores:
//
//   z[f][j] = sum_s Lambda[j][s] xi[f][s]
//
// with the operator stored DENSE -- the sparse fit's dropped entries are zeros -- for
// grids whose sample dimension S is small (cfg1-3, cfg5: S = 136..300, so a dense row
// costs a few times the kept entries but runs at tensor-core rate instead of FP32).
// Both operands are split into bf16 planes, x = hi + lo (16 significant bits), and
// three MMAs per k-step accumulate Ah.Bh + Ah.Bl + Al.Bh in fp32 TMEM (kind::f16).
// NumPy emulation at cfg3: 2.4e-6 normalized max error; a single bf16 / TF32 pass
// gives 1.1e-4 .. 1.9e-4, over the 1e-4 parity bar, so one pass is not an option.
//
// D = A . B^T: A = xi planes [F][S8] (M = 128 frames per tile), B = Lambda planes
// [J][S8] (N = 256 candidates per tile), both K-major with the 128-byte swizzle,
// k-blocks of 64 bf16.  Persistent CTAs (one per SM) walk the tiles; two TMEM
// accumulators (2 x 256 fp32 columns) let the epilogue of tile t overlap the MMAs of
// tile t+1.  Roles: warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA
// issuer, warps 2-5 epilogue (TMEM lane quarter = warp % 4, i.e. 32 frames each):
// tcgen05.ld 32 columns at a time, running per-frame argmax in registers (one
// atomicMax per frame per tile), z through a swizzled shared tile and a TMA store.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "tc_common.cuh"

namespace srpgpu {
namespace itc {

using namespace tc;

constexpr int IM = 128;   // frames per tile (TMEM lanes)
constexpr int IN = 256;   // candidates per tile (TMEM columns per accumulator)
constexpr int IK = 64;    // bf16 per k-block = 128 bytes = one swizzle atom row
constexpr int UK = 16;    // kind::f16 MMA K
// Two configurations: <2 stages, 4 epilogue warps> for operators with several k-blocks
// (SSPI / SI: MMA-bound), <1 stage, 8 epilogue warps> for a single k-block (the SLRI / LR
// candidate products, K = R or 2R: bound by the z write, so the epilogue gets twice the
// warps -- two per TMEM lane quarter, each draining half of the columns).
template <int NS, int kEpi>
struct __align__(1024) Smem {
  uint16_t a[NS][2][IM * IK];        // xi hi / lo, 16 KB per plane
  uint16_t b[NS][2][IN * IK];        // Lambda hi / lo, 32 KB per plane
  float stage[kEpi][2][32 * 32];     // z staging per epilogue warp, double-buffered, 4 KB
  uint64_t full[NS], empty[NS], tfull[2], tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int NS, int kEpi>
__global__ void __launch_bounds__(32 * (2 + kEpi), 1)
interp_tc_kernel(const __grid_constant__ CUtensorMap ma_hi, const __grid_constant__ CUtensorMap ma_lo,
                 const __grid_constant__ CUtensorMap mb_hi, const __grid_constant__ CUtensorMap mb_lo,
                 const __grid_constant__ CUtensorMap mz, int64_t F, int64_t J, int32_t nkb, float* __restrict__ z,
                 int32_t z_tma, unsigned long long* __restrict__ keys) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem<NS, kEpi>& sm =
      *reinterpret_cast<Smem<NS, kEpi>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (int)((F + IM - 1) / IM);
  const int n_tiles = (int)((J + IN - 1) / IN);
  const int total = m_tiles * n_tiles;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ma_hi);
    prefetch_tmap(&ma_lo);
    prefetch_tmap(&mb_hi);
    prefetch_tmap(&mb_lo);
    if (z_tma) prefetch_tmap(&mz);
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
    if (lane == 0) {
      constexpr uint32_t kBytes = 2u * (IM + IN) * IK * sizeof(uint16_t);
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int m_blk = tile % m_tiles, n_blk = tile / m_tiles;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % NS;
          mbar_wait(&sm.empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&sm.full[s], kBytes);
          tma_load_2d(sm.a[s][0], &ma_hi, &sm.full[s], kb * IK, m_blk * IM);
          tma_load_2d(sm.a[s][1], &ma_lo, &sm.full[s], kb * IK, m_blk * IM);
          tma_load_2d(sm.b[s][0], &mb_hi, &sm.full[s], kb * IK, n_blk * IN);
          tma_load_2d(sm.b[s][1], &mb_lo, &sm.full[s], kb * IK, n_blk * IN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::f16: D f32 (bits 4-5 = 1), A bf16 (7-9 = 1), B bf16 (10-12 = 1), both K-major
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(IN >> 3) << 17) |
                                 ((uint32_t)(IM >> 4) << 24);
      uint32_t g = 0, it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const uint32_t acc = it & 1;
        mbar_wait(&sm.tempty[acc], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * IN;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % NS;
          mbar_wait(&sm.full[s], (g / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ah = smem_desc(sm.a[s][0]), al = smem_desc(sm.a[s][1]);
          const uint64_t bh = smem_desc(sm.b[s][0]), bl = smem_desc(sm.b[s][1]);
#pragma unroll
          for (int k = 0; k < IK / UK; ++k) {
            const uint64_t off = (uint64_t)((k * UK * 2) >> 4);
            mma_bf16(d, ah + off, bh + off, idesc, (kb | k) != 0);
            mma_bf16(d, ah + off, bl + off, idesc, 1u);
            mma_bf16(d, al + off, bh + off, idesc, 1u);
          }
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull[acc]);
      }
    }
  } else {
    const int q = warp & 3;                          // TMEM lane quarter this warp may access
    const int e = warp - 2;                          // staging slot
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t stage0 = smem_u32(&sm.stage[e][0][0]);
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int m_blk = tile % m_tiles, n_blk = tile / m_tiles;
      const uint32_t acc = it & 1;
      mbar_wait(&sm.tfull[acc], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t f = (int64_t)m_blk * IM + q * 32 + lane;
      const int64_t j0 = (int64_t)n_blk * IN;
      const int64_t f0w = (int64_t)m_blk * IM + q * 32;       // first frame of this warp
      uint32_t best_ob = 0, best_j = 0;
      bool have = false;
      constexpr int kCpw = (IN / 32) / (kEpi / 4);   // 32-column chunks per epilogue warp
      const int c_lo = ((warp - 2) / 4) * kCpw;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + kCpw; ++c) {
        uint32_t r[32];
        tmem_ld32(lane_base + acc * IN + c * 32, r);
        const int64_t jc = j0 + c * 32;
        if (jc >= J) break;                          // warp-uniform
        // running argmax: ordered bits, strict '>' keeps the lowest index (np.argmax)
        if (jc + 32 <= J) {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const uint32_t ob = ordered_bits(__uint_as_float(r[t]));
            if (!have || ob > best_ob) { best_ob = ob; best_j = (uint32_t)(jc + t); have = true; }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const uint32_t ob = ordered_bits(__uint_as_float(r[t]));
            if (jc + t < J && (!have || ob > best_ob)) { best_ob = ob; best_j = (uint32_t)(jc + t); have = true; }
          }
        }
        if (z) {
          // the 32 x 32 block (rows = this warp's frames) goes through a 128-byte-swizzled
          // staging tile: TMA store when rows are 16-byte pitched, else coalesced row stores
          const uint32_t buf = stage0 + (uint32_t)(c & 1) * 4096u;
          if (z_tma && lane == 0) bulk_wait_read<1>();   // this buffer's previous store has read it
          __syncwarp();
          const uint32_t row = buf + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint32_t addr = row + (uint32_t)((ch ^ (lane & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r[4 * ch]), "r"(r[4 * ch + 1]),
                         "r"(r[4 * ch + 2]), "r"(r[4 * ch + 3])
                         : "memory");
          }
          if (z_tma) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&mz, &sm.stage[e][c & 1][0], (int)jc, (int)f0w);
              bulk_commit();
            }
          } else {
            __syncwarp();
            const bool col_ok = jc + lane < J;
            const uint32_t col = (uint32_t)((lane & 3) << 2);
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr) {
              const int64_t fr = f0w + rr;
              float v;
              asm volatile("ld.shared.f32 %0, [%1];"
                           : "=f"(v)
                           : "r"(buf + rr * 128 + (uint32_t)((((lane >> 2) ^ (rr & 7)) << 4)) + col)
                           : "memory");
              if (fr < F && col_ok) z[fr * J + jc + lane] = v;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty[acc]);
      if (keys && have && f < F)
        atomicMax(keys + f, ((unsigned long long)best_ob << 32) | (unsigned long long)(0xFFFFFFFFu - best_j));
    }
    if (lane == 0) bulk_wait_all();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// hi = bf16_rne(x), lo = bf16_rne(x - hi) into planes dst[0][r][c], dst[1][r][c] (pitch cols8),
// zero in [cols, cols8).  LAG_MAJOR: src[c * ld + r] (the map kernels' lag-major samples),
// else src[r * ld + c].  32 x 32 tiles through shared memory (coalesced both ways).
template <bool LAG_MAJOR>
__global__ void split_bf16_kernel(const float* __restrict__ src, int64_t ld, int64_t rows, int32_t cols,
                                  const int32_t* __restrict__ col_src, __nv_bfloat16* __restrict__ dst,
                                  int32_t cols8, int64_t r_base) {
  __shared__ float t[32][33];
  const int64_t r0 = r_base + (int64_t)blockIdx.y * 32;
  const int c0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    if (LAG_MAJOR) {   // t[c][r] = src[(c0 + k) * ld + r0 + tx]
      const int c = c0 + k;
      const int64_t r = r0 + tx;
      const int cs = (c < cols && col_src) ? __ldg(col_src + c) : c;
      t[k][tx] = (c < cols && r < rows) ? __ldg(src + (int64_t)cs * ld + r) : 0.f;
    } else {           // t[c][r] with r = r0 + k, c = c0 + tx
      const int c = c0 + tx;
      const int64_t r = r0 + k;
      const int cs = (c < cols && col_src) ? __ldg(col_src + c) : c;
      t[tx][k] = (c < cols && r < rows) ? __ldg(src + r * ld + cs) : 0.f;
    }
  }
  __syncthreads();
  const int64_t plane = rows * (int64_t)cols8;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k;
    const int c = c0 + tx;
    if (r < rows && c < cols8) {
      const float x = t[tx][k];
      const __nv_bfloat16 hi = __float2bfloat16_rn(x);
      const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
      dst[r * cols8 + c] = hi;
      dst[plane + r * cols8 + c] = lo;
    }
  }
}

// row-wise split: dst[p][r][c] = split(src[row_src[r]][c]) (lag-major samples -> lag-major
// planes, rows optionally permuted), rows [S], cols = frames
__global__ void split_rows_kernel(const float* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                                  const int32_t* __restrict__ row_src, __nv_bfloat16* __restrict__ dst,
                                  int64_t ld_dst, int64_t plane) {
  const int64_t r = blockIdx.y;
  const int64_t rs = row_src ? __ldg(row_src + r) : r;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    const float x = __ldg(src + rs * ld_src + c);
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    dst[r * ld_dst + c] = hi;
    dst[plane + r * ld_dst + c] = __float2bfloat16_rn(x - __bfloat162float(hi));
  }
}

// the same into fp32 TF32 hi / lo planes: hi = tf32_rne(x), lo = tf32_rne(x - hi)
__global__ void split_rows_tf32_kernel(const float* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                                       const int32_t* __restrict__ row_src, float* __restrict__ dst, int64_t ld_dst,
                                       int64_t plane) {
  const int64_t r = blockIdx.y;
  const int64_t rs = row_src ? __ldg(row_src + r) : r;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    const float x = __ldg(src + rs * ld_src + c);
    const float hi = tf32_rne(x);
    dst[r * ld_dst + c] = hi;
    dst[plane + r * ld_dst + c] = tf32_rne(x - hi);
  }
}

// the same into fp16 hi / lo planes: hi = f16_rne(s x), lo = f16_rne(s x - hi) (s: a power of
// two that keeps the operand in fp16 range; 11 + 11 significant bits, as the TF32 split)
__global__ void split_rows_f16_kernel(const float* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                                      const int32_t* __restrict__ row_src, float scale, __half* __restrict__ dst,
                                      int64_t ld_dst, int64_t plane) {
  const int64_t r = blockIdx.y;
  const int64_t rs = row_src ? __ldg(row_src + r) : r;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    const float x = __ldg(src + rs * ld_src + c) * scale;
    const __half hi = __float2half_rn(x);
    dst[r * ld_dst + c] = hi;
    dst[plane + r * ld_dst + c] = __float2half_rn(x - __half2float(hi));
  }
}

}  // namespace itc

int reset_keys(uint64_t* keys, int64_t F, cudaStream_t st);

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_split_bf16_cols(const float* src, int64_t ld_src, int32_t lag_major, int64_t rows, int32_t cols,
                                      const int32_t* col_src, void* dst, int32_t cols8, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rows >= 0 && cols >= 0 && cols8 >= cols && cols8 % 8 == 0, SRPGPU_ERR_DIMENSION,
                   "split_bf16: bad shape (rows %lld, cols %d, cols8 %d)", (long long)rows, cols, cols8);
  SRPGPU_CHECK_ARG(lag_major ? ld_src >= rows : ld_src >= cols, SRPGPU_ERR_DIMENSION, "split_bf16: bad pitch");
  SRPGPU_CHECK_ARG(((uintptr_t)dst & 15) == 0, SRPGPU_ERR_VALUE, "split_bf16: destination must be 16-byte aligned");
  if (rows == 0 || cols8 == 0) return SRPGPU_OK;
  const int64_t yb = (rows + 31) / 32;
  cudaStream_t st = as_stream(stream);
  auto* d = reinterpret_cast<__nv_bfloat16*>(dst);
  for (int64_t y0 = 0; y0 < yb; y0 += 65535) {   // grid.y limit: launch in row chunks
    dim3 grid((unsigned)((cols8 + 31) / 32), (unsigned)std::min<int64_t>(65535, yb - y0)), block(32, 8);
    if (lag_major)
      itc::split_bf16_kernel<true><<<grid, block, 0, st>>>(src, ld_src, rows, cols, col_src, d, cols8, y0 * 32);
    else
      itc::split_bf16_kernel<false><<<grid, block, 0, st>>>(src, ld_src, rows, cols, col_src, d, cols8, y0 * 32);
    SRPGPU_CHECK_LAUNCH("split_bf16");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_split_bf16_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                                      const int32_t* row_src, void* dst, int64_t ld_dst, int64_t rows_dst,
                                      srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rows >= 0 && cols >= 0 && ld_src >= cols && ld_dst >= cols && rows_dst >= rows, SRPGPU_ERR_DIMENSION,
                   "split_bf16_rows: bad shape");
  SRPGPU_CHECK_ARG(((uintptr_t)dst & 15) == 0, SRPGPU_ERR_VALUE, "split_bf16_rows: destination must be 16-byte aligned");
  if (rows == 0 || cols == 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>((cols + 255) / 256, 64), (unsigned)nr);
    itc::split_rows_kernel<<<grid, 256, 0, st>>>(row_src ? src : src + r0 * ld_src, ld_src, nr, cols,
                                                 row_src ? row_src + r0 : nullptr,
                                                 reinterpret_cast<__nv_bfloat16*>(dst) + r0 * ld_dst, ld_dst,
                                                 rows_dst * ld_dst);
    SRPGPU_CHECK_LAUNCH("split_bf16_rows");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_split_tf32_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                                      const int32_t* row_src, float* dst, int64_t ld_dst, int64_t rows_dst,
                                      srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rows >= 0 && cols >= 0 && ld_src >= cols && ld_dst >= cols && rows_dst >= rows, SRPGPU_ERR_DIMENSION,
                   "split_tf32_rows: bad shape");
  SRPGPU_CHECK_ARG(((uintptr_t)dst & 15) == 0, SRPGPU_ERR_VALUE, "split_tf32_rows: destination must be 16-byte aligned");
  if (rows == 0 || cols == 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>((cols + 255) / 256, 64), (unsigned)nr);
    itc::split_rows_tf32_kernel<<<grid, 256, 0, st>>>(row_src ? src : src + r0 * ld_src, ld_src, nr, cols,
                                                      row_src ? row_src + r0 : nullptr, dst + r0 * ld_dst, ld_dst,
                                                      rows_dst * ld_dst);
    SRPGPU_CHECK_LAUNCH("split_tf32_rows");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_split_f16_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols,
                                     const int32_t* row_src, float scale, void* dst, int64_t ld_dst,
                                     int64_t rows_dst, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rows >= 0 && cols >= 0 && ld_src >= cols && ld_dst >= cols && rows_dst >= rows, SRPGPU_ERR_DIMENSION,
                   "split_f16_rows: bad shape");
  SRPGPU_CHECK_ARG(((uintptr_t)dst & 15) == 0, SRPGPU_ERR_VALUE, "split_f16_rows: destination must be 16-byte aligned");
  if (rows == 0 || cols == 0) return SRPGPU_OK;
  cudaStream_t st = as_stream(stream);
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>((cols + 255) / 256, 64), (unsigned)nr);
    itc::split_rows_f16_kernel<<<grid, 256, 0, st>>>(row_src ? src : src + r0 * ld_src, ld_src, nr, cols,
                                                     row_src ? row_src + r0 : nullptr, scale,
                                                     reinterpret_cast<__half*>(dst) + r0 * ld_dst, ld_dst,
                                                     rows_dst * ld_dst);
    SRPGPU_CHECK_LAUNCH("split_f16_rows");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_split_bf16(const float* src, int64_t ld_src, int32_t lag_major, int64_t rows, int32_t cols,
                                 void* dst, int32_t cols8, srpgpu_stream_t stream) {
  return srpgpu_split_bf16_cols(src, ld_src, lag_major, rows, cols, nullptr, dst, cols8, stream);
}

extern "C" int srpgpu_interp_map_tc(const void* samples_planes, int64_t num_frames, const void* op_planes,
                                    int64_t num_candidates, int32_t cols8, float* z, uint64_t* keys,
                                    srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_frames >= 0 && num_candidates >= 1 && cols8 >= 8 && cols8 % 8 == 0, SRPGPU_ERR_DIMENSION,
                   "interp_map_tc: bad shape (frames %lld, candidates %lld, cols8 %d)", (long long)num_frames,
                   (long long)num_candidates, cols8);
  SRPGPU_CHECK_ARG(((uintptr_t)samples_planes & 15) == 0 && ((uintptr_t)op_planes & 15) == 0, SRPGPU_ERR_VALUE,
                   "interp_map_tc: operands must be 16-byte aligned");
  SRPGPU_CHECK_ARG(num_frames < (1ll << 31) && num_candidates < (1ll << 31), SRPGPU_ERR_DIMENSION,
                   "interp_map_tc: too many frames / candidates");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames == 0) return SRPGPU_OK;
  using namespace itc;
  const auto* xa = reinterpret_cast<const uint16_t*>(samples_planes);
  const auto* xb = reinterpret_cast<const uint16_t*>(op_planes);
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo, mz;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if ((s = make_map_2d(&ma_hi, bf, 2, xa, num_frames, cols8, cols8, IK, IM, "interp_map_tc")) ||
      (s = make_map_2d(&ma_lo, bf, 2, xa + num_frames * cols8, num_frames, cols8, cols8, IK, IM, "interp_map_tc")) ||
      (s = make_map_2d(&mb_hi, bf, 2, xb, num_candidates, cols8, cols8, IK, IN, "interp_map_tc")) ||
      (s = make_map_2d(&mb_lo, bf, 2, xb + num_candidates * cols8, num_candidates, cols8, cols8, IK, IN,
                       "interp_map_tc")))
    return s;
  // z through TMA stores needs 16-byte row pitches (J % 4 == 0) and a 16-byte base
  const int z_tma = (z != nullptr && num_candidates % 4 == 0 && ((uintptr_t)z & 15) == 0) ? 1 : 0;
  mz = ma_hi;
  if (z_tma && (s = make_map_2d(&mz, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, z, num_frames, num_candidates,
                                num_candidates, 32, 32, "interp_map_tc")))
    return s;
  const int64_t tiles = ((num_frames + IM - 1) / IM) * ((num_candidates + IN - 1) / IN);
  SRPGPU_CHECK_ARG(tiles < (1ll << 31), SRPGPU_ERR_DIMENSION, "interp_map_tc: too many tiles");
  const int nkb = (cols8 + IK - 1) / IK;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, num_sms());
  auto run = [&](auto kern, size_t smem, int threads) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      set_error("interp_map_tc: cannot reserve %zu B shared memory", smem);
      return SRPGPU_ERR_LAUNCH;
    }
    kern<<<grid, threads, smem, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, mz, num_frames, num_candidates, nkb, z, z_tma,
                                      reinterpret_cast<unsigned long long*>(keys));
    return SRPGPU_OK;
  };
  // one k-block (the low-rank candidate products): z-write bound -> 8 epilogue warps
  s = nkb == 1 ? run(interp_tc_kernel<1, 8>, sizeof(Smem<1, 8>) + 1024, 32 * (2 + 8))
               : run(interp_tc_kernel<2, 4>, sizeof(Smem<2, 4>) + 1024, 32 * (2 + 4));
  if (s) return s;
  SRPGPU_CHECK_LAUNCH("interp_map_tc");
  return SRPGPU_OK;
}
