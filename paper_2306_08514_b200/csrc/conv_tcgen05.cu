// Conventional SRP map on the 5th-generation tensor cores (sm_100a):
//
//   z[f][i] = 2 Re( sum_k H[i][k] psi[f][k] )          srp.py:65-71
//           = 2 * sum_k' A[i][k'] B[f][k']
//   A = interleaved (Re H, -Im H) rows  [J][2PB]   (fp32 storage, read as TF32)
//   B = psi viewed as interleaved (re, im) floats [F][2PB]
//
// D = A . B^T is a K-major x K-major ("TN") GEMM with M = candidates, N = frames.
// Warp-specialised CTA (192 threads):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D tiles of A and B into a
//               STAGES-deep shared-memory ring (128-byte swizzle), mbarrier
//               full/empty handshake;
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::tf32, accumulator in TMEM,
//               tcgen05.commit frees each smem stage and finally signals the
//               epilogue;
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers, x2, coalesced store
//               of z[f][i] (lanes = consecutive candidates) and the fused
//               per-frame argmax (packed keys, atomicMax).
// Tiles are rasterised in groups of GROUP_M candidate tiles so concurrently
// running CTAs share both A and B k-slices in L2.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"

namespace srpgpu {
namespace tc {

constexpr int BLOCK_M = 128;
constexpr int BLOCK_K = 32;          // fp32 elements = 128 bytes = one swizzle atom row
constexpr int UMMA_K = 8;            // tf32: 32 bytes per MMA
constexpr int STAGES = 4;
constexpr int GROUP_M = 16;
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// K-major operand tile, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;          // start address
  d |= (uint64_t)1 << 16;                  // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BLOCK_N>
struct __align__(1024) Smem {
  float a[STAGES][BLOCK_M * BLOCK_K];   // 16 KB per stage
  float b[STAGES][BLOCK_N * BLOCK_K];   // 16 / 32 KB per stage
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full;
  uint32_t tmem_base;
};

// On-chip steering operand: A[i][2c] = cos(theta), A[i][2c+1] = -sin(theta) with
// theta = pi k x[i][p] / K for complex column c = p (K-1) + k - 1 (srp.py:51-62,
// frontend.py:67-71), x = dt * fs.  Generated per k-block by the four epilogue warps
// (one row each: a sincospi seed per pair segment, then a complex rotation per bin),
// rounded to TF32 and written in the 128-byte-swizzled K-major layout TMA would produce.
struct GenParams {
  const float* xtab;   // [J][P]
  int32_t P;
  int32_t B;           // bins per pair (K - 1)
  float inv_k;         // 1 / K
};

// round to nearest TF32 in one instruction (ties away from zero; the phasors never tie in
// practice, and rounding-to-nearest keeps the product unbiased unlike plain truncation)
__device__ __forceinline__ uint32_t cvt_tf32(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return u;
}

// Per-row generator state carried across k-blocks (one thread per operand row).
struct GenState {
  int pair;          // pair of the carried rotation (-1: none)
  int next_k;        // bin whose phasor `seed` holds
  int since;         // blocks since the last exact seed
  float2 seed, s1, s2, s4, s8;   // exp(j pi k x / K) at next_k, and step powers
  float x;
};

__device__ __forceinline__ void gen_state_init(GenState& g) {
  g.pair = -1; g.next_k = 0; g.since = 0; g.x = 0.f;
  g.seed = g.s1 = g.s2 = g.s4 = g.s8 = make_float2(1.f, 0.f);
}

__device__ __forceinline__ void gen_a_block(float* a_stage, int row, int64_t i, bool valid, int kb,
                                            const GenParams& gp, GenState& g) {
  const int total = gp.P * gp.B;
  const int c0 = kb * 16;
  float2 e[16];
  const int p0 = c0 / gp.B, p1 = (c0 + 15) / gp.B;
  if (valid && p0 == p1 && c0 + 15 < total) {
    // fast path: 16 consecutive bins of one pair, e_j = seed * step^j (depth-4 product tree)
    const int k0 = c0 - p0 * gp.B + 1;
    if (g.pair != p0 || g.next_k != k0 || g.since >= 4) {
      if (g.pair != p0) {
        g.pair = p0;
        g.x = __ldg(gp.xtab + i * gp.P + p0);
        float sn, cs;
        sincospif(g.x * gp.inv_k, &sn, &cs);
        g.s1 = make_float2(cs, sn);
        g.s2 = cmul(g.s1, g.s1);
        g.s4 = cmul(g.s2, g.s2);
        g.s8 = cmul(g.s4, g.s4);
      }
      float sn, cs;
      sincospif((float)k0 * g.x * gp.inv_k, &sn, &cs);   // exact re-seed bounds the drift
      g.seed = make_float2(cs, sn);
      g.since = 0;
    }
    e[0] = g.seed;
    e[1] = cmul(e[0], g.s1);
    e[2] = cmul(e[0], g.s2);
    e[3] = cmul(e[1], g.s2);
#pragma unroll
    for (int j = 0; j < 4; ++j) e[4 + j] = cmul(e[j], g.s4);
#pragma unroll
    for (int j = 0; j < 8; ++j) e[8 + j] = cmul(e[j], g.s8);
    g.seed = cmul(e[8], g.s8);
    g.next_k = k0 + 16;
    g.since += 1;
  } else {
    // block straddles a pair boundary (or the tail): exact phasor per element
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = c0 + j;
      e[j] = make_float2(0.f, 0.f);
      if (valid && c < total) {
        const int pc = c / gp.B;
        const int k = c - pc * gp.B + 1;
        const float x = __ldg(gp.xtab + i * gp.P + pc);
        float sn, cs;
        sincospif((float)k * x * gp.inv_k, &sn, &cs);
        e[j] = make_float2(cs, sn);
      }
    }
    g.pair = -1;
  }
  unsigned char* rowp = reinterpret_cast<unsigned char*>(a_stage) + row * 128;
#pragma unroll
  for (int q = 0; q < 8; ++q)   // (Re H, -Im H), TF32-rounded, 128-byte swizzle: chunk q -> q ^ (row & 7)
    *reinterpret_cast<uint4*>(rowp + ((q ^ (row & 7)) << 4)) =
        make_uint4(cvt_tf32(e[2 * q].x), cvt_tf32(-e[2 * q].y), cvt_tf32(e[2 * q + 1].x),
                   cvt_tf32(-e[2 * q + 1].y));
}

template <int BLOCK_N, bool GEN_A>
__global__ void __launch_bounds__(kThreads, 1)
conv_tf32_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 int64_t J, int64_t F, int32_t Kd, float* __restrict__ z,
                 unsigned long long* __restrict__ keys, float alpha, const GenParams gp) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzled tiles
  Smem<BLOCK_N>& sm = *reinterpret_cast<Smem<BLOCK_N>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // grouped rasterisation: GROUP_M m-tiles share each n-tile sweep
  const int m_tiles = (int)((J + BLOCK_M - 1) / BLOCK_M);
  const int n_tiles = (int)((F + BLOCK_N - 1) / BLOCK_N);
  const int tile = blockIdx.x;
  const int group = tile / (GROUP_M * n_tiles);
  const int first_m = group * GROUP_M;
  const int gsize = min(m_tiles - first_m, GROUP_M);
  const int m_blk = first_m + (tile % (GROUP_M * n_tiles)) % gsize;
  const int n_blk = (tile % (GROUP_M * n_tiles)) / gsize;
  const int num_kb = (Kd + BLOCK_K - 1) / BLOCK_K;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], GEN_A ? 1 + 128 : 1);   // + the 128 generator threads
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "n"(BLOCK_N < 32 ? 32 : BLOCK_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t kBytes = ((GEN_A ? 0 : BLOCK_M) + BLOCK_N) * BLOCK_K * sizeof(float);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t round = kb / STAGES;
        mbar_wait(&sm.empty[s], (round & 1) ^ 1);
        mbar_expect_tx(&sm.full[s], kBytes);
        if (!GEN_A) tma_load_2d(sm.a[s], &map_a, &sm.full[s], kb * BLOCK_K, m_blk * BLOCK_M);
        tma_load_2d(sm.b[s], &map_b, &sm.full[s], kb * BLOCK_K, n_blk * BLOCK_N);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::tf32: D f32 (bits 4-5 = 1), A/B tf32 (= 2), both K-major, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BLOCK_N >> 3) << 17) |
                             ((uint32_t)(BLOCK_M >> 4) << 24);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t round = kb / STAGES;
        mbar_wait(&sm.full[s], round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = smem_desc(sm.a[s]);
        const uint64_t db = smem_desc(sm.b[s]);
#pragma unroll
        for (int k = 0; k < BLOCK_K / UMMA_K; ++k) {
          // advance the start address by k * 32 bytes inside the 128-byte swizzle row
          mma_tf32(tmem, da + (uint64_t)((k * UMMA_K * 4) >> 4), db + (uint64_t)((k * UMMA_K * 4) >> 4),
                   idesc, (kb | k) != 0);
        }
        mma_commit(&sm.empty[s]);
      }
      mma_commit(&sm.tmem_full);
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarter (warp % 4)
    const int quarter = warp & 3;
    if (GEN_A) {   // generate the steering operand stage by stage
      const int row = quarter * 32 + lane;
      const int64_t gi = (int64_t)m_blk * BLOCK_M + row;
      GenState g;
      gen_state_init(g);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t round = kb / STAGES;
        mbar_wait(&sm.empty[s], (round & 1) ^ 1);
        gen_a_block(sm.a[s], row, gi, gi < J, kb, gp, g);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.full[s])) : "memory");
      }
    }
    mbar_wait(&sm.tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int64_t i = (int64_t)m_blk * BLOCK_M + quarter * 32 + lane;
    const bool row_ok = i < J;
#pragma unroll 1
    for (int c0 = 0; c0 < BLOCK_N; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, r);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int64_t f = (int64_t)n_blk * BLOCK_N + c0 + c;
        if (f >= F) break;
        const float v = alpha * __uint_as_float(r[c]);
        if (z && row_ok) z[f * J + i] = v;
        if (keys) {
          unsigned long long k = row_ok ? make_key(v, (uint32_t)i) : 0ull;
          k = warp_key_max(k);
          if (lane == 0 && k) atomicMax(keys + f, k);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(BLOCK_N < 32 ? 32 : BLOCK_N));
  }
}

// ---- host: TMA descriptors through the driver entry point (no -lcuda) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("srp_map_tc: cuTensorMapEncodeTiled unavailable");
    return SRPGPU_ERR_LAUNCH;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)BLOCK_K, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  static const int tma_tf32 = [] {
    const char* e = getenv("SRPGPU_TMA_TF32");
    return e && e[0] == '1';
  }();
  CUresult r = enc(map, tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("srp_map_tc: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SRPGPU_ERR_LAUNCH;
  }
  return SRPGPU_OK;
}

template <int BLOCK_N, bool GEN_A>
static int launch(const float* gcc, int64_t gcc_ld, int64_t F, int32_t Kd, const float* h2, int64_t h2_ld,
                  int64_t J, float* z, uint64_t* keys, cudaStream_t st, const GenParams& gp) {
  CUtensorMap ma, mb;
  int s = make_map(&mb, gcc, F, Kd, gcc_ld, BLOCK_N);
  if (s) return s;
  if (GEN_A) ma = mb;
  else if ((s = make_map(&ma, h2, J, Kd, h2_ld, BLOCK_M))) return s;
  const size_t smem = sizeof(Smem<BLOCK_N>) + 1024;
  auto kern = conv_tf32_kernel<BLOCK_N, GEN_A>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("srp_map_tc: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  const int64_t tiles = ((J + BLOCK_M - 1) / BLOCK_M) * ((F + BLOCK_N - 1) / BLOCK_N);
  SRPGPU_CHECK_ARG(tiles < (1ll << 31), SRPGPU_ERR_DIMENSION, "srp_map_tc: too many tiles");
  kern<<<(unsigned)tiles, kThreads, smem, st>>>(ma, mb, J, F, Kd, z,
                                                 reinterpret_cast<unsigned long long*>(keys), 2.0f, gp);
  SRPGPU_CHECK_LAUNCH("srp_map_tc");
  return SRPGPU_OK;
}

// Round-to-nearest-even to TF32 (10-bit mantissa), so the tensor-core product is
// unbiased (plain fp32 bits are truncated by kind::tf32).  Also re-pitches rows.
__global__ void round_tf32_kernel(const float* __restrict__ src, int64_t ld_src, float* __restrict__ dst,
                                 int64_t ld_dst, int64_t rows, int64_t cols) {
  const int64_t r = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ld_dst;
       c += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (c < cols) v = tf32_rne(__ldg(src + r * ld_src + c));
    dst[r * ld_dst + c] = v;
  }
}

}  // namespace tc

int reset_keys(uint64_t* keys, int64_t F, cudaStream_t st);

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_round_tf32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst,
                                 int64_t rows, int64_t cols, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(ld_dst >= cols && ld_src >= cols && rows >= 0, SRPGPU_ERR_DIMENSION,
                   "round_tf32: bad pitches");
  if (rows == 0 || ld_dst == 0) return SRPGPU_OK;
  SRPGPU_CHECK_ARG(rows <= 65535ll * 1024, SRPGPU_ERR_DIMENSION, "round_tf32: too many rows");
  const int64_t done_rows = 0;
  (void)done_rows;
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>((ld_dst + 255) / 256, 64), (unsigned)nr);
    tc::round_tf32_kernel<<<grid, 256, 0, as_stream(stream)>>>(src + r0 * ld_src, ld_src, dst + r0 * ld_dst,
                                                                ld_dst, nr, cols);
    SRPGPU_CHECK_LAUNCH("round_tf32");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_srp_map_tc(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t gcc_len,
                                 const float* h2, int64_t h2_ld, int64_t num_candidates, float* z,
                                 uint64_t* keys, srpgpu_stream_t stream) {
  const int32_t Kd = 2 * gcc_len;
  SRPGPU_CHECK_ARG(gcc_len >= 1 && num_candidates >= 1, SRPGPU_ERR_DIMENSION, "srp_map_tc: empty operator");
  SRPGPU_CHECK_ARG(gcc_ld >= Kd && h2_ld >= Kd && gcc_ld % 4 == 0 && h2_ld % 4 == 0, SRPGPU_ERR_VALUE,
                   "srp_map_tc: row pitches must cover 2*gcc_len floats and be 16-byte multiples");
  SRPGPU_CHECK_ARG(((uintptr_t)gcc & 15) == 0 && ((uintptr_t)h2 & 15) == 0, SRPGPU_ERR_VALUE,
                   "srp_map_tc: operands must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames <= 0) return SRPGPU_OK;
  const int64_t m_tiles = (num_candidates + tc::BLOCK_M - 1) / tc::BLOCK_M;
  const int64_t n256 = (num_frames + 255) / 256;
  const tc::GenParams gp = {};
  if (m_tiles * n256 >= 2 * (int64_t)num_sms())
    return tc::launch<256, false>(gcc, gcc_ld, num_frames, Kd, h2, h2_ld, num_candidates, z, keys, st, gp);
  return tc::launch<128, false>(gcc, gcc_ld, num_frames, Kd, h2, h2_ld, num_candidates, z, keys, st, gp);
}

extern "C" int srpgpu_srp_map_tdoa(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t num_pairs,
                                   int32_t half_len, const float* xtab, int64_t num_candidates, float* z,
                                   uint64_t* keys, srpgpu_stream_t stream) {
  const int32_t bins = half_len - 1;
  const int32_t Kd = 2 * num_pairs * bins;
  SRPGPU_CHECK_ARG(num_pairs >= 1 && bins >= 1 && num_candidates >= 1, SRPGPU_ERR_DIMENSION,
                   "srp_map_tdoa: empty operator");
  SRPGPU_CHECK_ARG(gcc_ld >= Kd && gcc_ld % 4 == 0 && ((uintptr_t)gcc & 15) == 0, SRPGPU_ERR_VALUE,
                   "srp_map_tdoa: gcc rows must cover 2*P*(K-1) floats with a 16-byte pitch");
  cudaStream_t st = as_stream(stream);
  int s = reset_keys(keys, num_frames, st);
  if (s) return s;
  if (num_frames <= 0) return SRPGPU_OK;
  tc::GenParams gp;
  gp.xtab = xtab; gp.P = num_pairs; gp.B = bins; gp.inv_k = 1.0f / (float)half_len;
  const int64_t m_tiles = (num_candidates + tc::BLOCK_M - 1) / tc::BLOCK_M;
  const int64_t n256 = (num_frames + 255) / 256;
  if (m_tiles * n256 >= 2 * (int64_t)num_sms())
    return tc::launch<256, true>(gcc, gcc_ld, num_frames, Kd, nullptr, 0, num_candidates, z, keys, st, gp);
  return tc::launch<128, true>(gcc, gcc_ld, num_frames, Kd, nullptr, 0, num_candidates, z, keys, st, gp);
}
