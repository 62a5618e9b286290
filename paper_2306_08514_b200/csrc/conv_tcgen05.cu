// Conventional SRP map on the 5th-generation tensor cores (sm_100a):
//
//   z[f][i] = 2 Re( sum_k H[i][k] psi[f][k] )          srp.py:65-71
//           = 2 * sum_k' A[i][k'] B[f][k']
//   A = interleaved (Re H, -Im H) rows  [J][2PB]   (TF32 operands)
//   B = psi viewed as interleaved (re, im) floats [F][2PB]
//
// D = A . B^T is a K-major x K-major ("TN") GEMM with M = candidates (128 per CTA),
// N = frames (256 per CTA), tcgen05.mma.cta_group::1.kind::tf32 with the accumulator in
// TMEM.  A is either streamed by TMA from a stored matrix (srpgpu_srp_map_tc, the
// drop-in SrpMatrix) or generated on chip from the TDOA table (srpgpu_srp_map_tdoa:
// the steering matrix of a large grid is never stored).  K is accumulated in chunks
// folded into fp32 registers (see conv_gen_chunked_kernel) because the tensor core's
// in-pipe accumulation is not IEEE fp32.  Epilogue: coalesced z stores and the fused
// per-frame argmax (packed keys, atomicMax).  Tiles are rasterised in groups of
// GROUP_M candidate tiles so concurrently running CTAs share k-slices in L2.
#include "tc_common.cuh"

namespace srpgpu {
namespace tc {

constexpr int BLOCK_M = 128;
constexpr int BLOCK_K = 32;          // fp32 elements = 128 bytes = one swizzle atom row
constexpr int UMMA_K = 8;            // tf32: 32 bytes per MMA
constexpr int GROUP_M = 16;

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

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

// Round a finite fp32 value to nearest TF32, ties away from zero (= cvt.rna.tf32.f32,
// which sm_100a emulates in ~5 instructions): add half a TF32 ulp to the magnitude bits
// (sign-magnitude format: the carry rounds |x| up and propagates into the exponent) and
// clear the 13 dropped bits.  The phasors are bounded by 1, so no overflow to inf.
// Rounding to nearest keeps the product unbiased, unlike the tensor core's truncation.
__device__ __forceinline__ uint32_t cvt_tf32(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
}

// the same rounding for an MMA operand only: kind::tf32 ignores the low 13 bits, so the
// mask is not needed (one instruction)
__device__ __forceinline__ uint32_t cvt_tf32_op(float x) { return __float_as_uint(x) + 0x1000u; }

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Per-thread generator state carried across k-blocks: the (pair, bin) position of the
// thread's first bin in the current block is advanced incrementally (no integer
// division in the loop), and the phasor rotation of the current pair is carried.
struct GenState {
  int p;             // pair of the first bin of this thread's 8 in the current k-block
  int k;             // its bin (1-based, <= B)
  int seeded_p;      // pair of the carried rotation (-1: none)
  int since;         // blocks since the last exact seed
  float2 seed, s1, s2, s4, s16;  // exp(j pi k x / K) at bin k of pair p, and step powers
  float x;
};

__device__ __forceinline__ void gen_state_init(GenState& g, int c0, int B) {
  g.p = c0 / B;
  g.k = c0 - g.p * B + 1;
  g.seeded_p = -1; g.since = 0; g.x = 0.f;
  g.seed = g.s1 = g.s2 = g.s4 = g.s16 = make_float2(1.f, 0.f);
}

// The GEMM kernel (128 candidates x 256 frames per CTA).  The tensor core's in-pipe
// accumulation is not IEEE fp32 (measured: 3.8e-5 normalized error against an exact
// evaluation of its own TF32 operands at K = 3600), so K is cut into chunks of CHUNK
// k-blocks accumulated in two alternating 256-column TMEM tiles (all 512 columns);
// while the MMA fills one, eight folding warps tcgen05.ld the other and add it into
// fp32 running sums held in registers.  With SPLIT the three 3xTF32 products go to the
// same chunk tile.  Roles (20 warps): warpgroup 0 = control (warp 0 TMA of psi, and
// of A when GEN = false; warp 1 TMEM alloc + MMA issue), shrunk to kCtlRegs registers;
// warps 4..19 = steering generators (four threads per operand row, 4 bins each) and
// folders: warp w owns TMEM lane quarter w % 4 and column quarter (w - 4) / 4, 64
// running sums per thread, grown to kWorkerRegs registers.  Sixteen worker warps hide
// the generator's per-block latency (it is a serial wait/generate/fence/arrive chain
// per warp) far better than eight warps holding 128 sums each.
constexpr int CHUNK = 16;
constexpr int kCtl = 4;                            // control warpgroup: 0 TMA, 1 MMA, 2-3 idle
constexpr int kWorkers = 16;                       // generator + fold warps (4 warpgroups)
constexpr int kThreadsC = 32 * (kCtl + kWorkers);
// setmaxnreg redistributes the CTA's own pool (launch: 640 threads x 96 registers):
// 4 warps x 32 + 16 warps x 112 = 61440 registers exactly (inc blocks if over)
constexpr int kCtlRegs = 32, kWorkerRegs = 112;
static_assert(32 * (kCtl * kCtlRegs + kWorkers * kWorkerRegs) <= kThreadsC * 96, "register pool");
constexpr int kNB = 16 * BLOCK_M / (32 * kWorkers); // bins per generator thread per k-block
constexpr int kFoldCols = 256 / (kWorkers / 4);     // accumulator columns per fold thread

template <bool SPLIT>
struct __align__(1024) SmemC {
  static constexpr int BN = 256;
  static constexpr int NS = SPLIT ? 2 : 4;
  static constexpr int NP = SPLIT ? 2 : 1;
  float a[NS][NP][BLOCK_M * BLOCK_K];
  float b[NS][NP][BN * BLOCK_K];
  uint64_t full[NS];
  uint64_t empty[NS];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// NB bins [NB part, NB part + NB) of the current k-block for one operand row.  The row
// holds the conjugate phasors exp(-j pi k x / K) as (re, im) = (cos, -sin) pairs.  Fast
// path: product tree from a carried seed, re-seeded exactly every kReseed blocks and at
// pair changes; a block straddling a pair boundary (or past the last pair) takes the
// compact per-bin path.  Advances g.
constexpr int kReseed = 8;

template <bool SPLIT>
__device__ __forceinline__ void store4(uint32_t hi_addr, uint32_t lo_addr, float v0, float v1, float v2, float v3) {
  if (SPLIT) {
    const uint32_t h0 = cvt_tf32(v0), h1 = cvt_tf32(v1), h2 = cvt_tf32(v2), h3 = cvt_tf32(v3);
    sts128(hi_addr, h0, h1, h2, h3);
    sts128(lo_addr, cvt_tf32_op(v0 - __uint_as_float(h0)), cvt_tf32_op(v1 - __uint_as_float(h1)),
           cvt_tf32_op(v2 - __uint_as_float(h2)), cvt_tf32_op(v3 - __uint_as_float(h3)));
  } else {
    sts128(hi_addr, cvt_tf32_op(v0), cvt_tf32_op(v1), cvt_tf32_op(v2), cvt_tf32_op(v3));
  }
}

template <bool SPLIT, int NB>
__device__ __forceinline__ void gen_a_part(uint32_t rowp, uint32_t rowl, const uint32_t (&off)[NB / 2], int qbase,
                                           int rx, int64_t i, const GenParams& gp, GenState& g) {
  static_assert(NB == 4 || NB == 8, "bins per thread");
  if (g.p < gp.P && g.k + NB - 1 <= gp.B) {
    if (g.seeded_p != g.p || g.since >= kReseed) {
      if (g.seeded_p != g.p) {
        g.seeded_p = g.p;
        g.x = __ldg(gp.xtab + i * gp.P + g.p);
        float sn, cs;
        sincospif(g.x * gp.inv_k, &sn, &cs);
        g.s1 = make_float2(cs, -sn);
        g.s2 = cmul(g.s1, g.s1);
        g.s4 = cmul(g.s2, g.s2);
        const float2 s8 = cmul(g.s4, g.s4);
        g.s16 = cmul(s8, s8);                          // step to the next block
      }
      float sn, cs;
      sincospif((float)g.k * g.x * gp.inv_k, &sn, &cs);
      g.seed = make_float2(cs, -sn);
      g.since = 0;
    }
    float2 e[NB];
    e[0] = g.seed;
    e[1] = cmul(e[0], g.s1);
    e[2] = cmul(e[0], g.s2);
    e[3] = cmul(e[1], g.s2);
    if (NB == 8) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[4 + j] = cmul(e[j], g.s4);
    }
    g.seed = cmul(e[0], g.s16);
    g.since += 1;
#pragma unroll
    for (int qq = 0; qq < NB / 2; ++qq)
      store4<SPLIT>(rowp + off[qq], rowl + off[qq], e[2 * qq].x, e[2 * qq].y, e[2 * qq + 1].x, e[2 * qq + 1].y);
  } else {
    int pp = g.p, kk = g.k;
#pragma unroll 1
    for (int j = 0; j < NB; j += 2) {
      float v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float sn = 0.f, cs = 0.f;
        if (pp < gp.P) sincospif((float)kk * __ldg(gp.xtab + i * gp.P + pp) * gp.inv_k, &sn, &cs);
        v[2 * h] = cs;
        v[2 * h + 1] = -sn;
        if (++kk > gp.B) { kk = 1; ++pp; }
      }
      const uint32_t o = (uint32_t)(((qbase + j / 2) ^ rx) << 4);
      store4<SPLIT>(rowp + o, rowl + o, v[0], v[1], v[2], v[3]);
    }
    g.seeded_p = -1;
  }
  g.k += 16;                                            // B >= 16 (checked on the host)
  if (g.k > gp.B) { g.k -= gp.B; ++g.p; }
}

// GEN = false: the steering operand is streamed by TMA from a stored matrix instead
// (map_a), with the same chunked accumulation (the drop-in SrpMatrix path).
template <bool SPLIT, bool GEN = true>
__global__ void __launch_bounds__(kThreadsC, 1)
conv_gen_chunked_kernel(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_b2,
                        const __grid_constant__ CUtensorMap map_a, int64_t J, int64_t F, int32_t Kd,
                        float* __restrict__ z, unsigned long long* __restrict__ keys, float alpha,
                        const GenParams gp, int32_t ksplit, float* __restrict__ zpart) {
  constexpr int BN = 256;
  using SM = SmemC<SPLIT>;
  constexpr int NS = SM::NS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (int)((J + BLOCK_M - 1) / BLOCK_M);
  const int n_tiles = (int)((F + BN - 1) / BN);
  // split-K (small grids): CTA = (output tile, K slice); K slices are whole chunks
  const int ks = blockIdx.x % ksplit;
  const int tile = blockIdx.x / ksplit;
  // raster: with a stored operator, groups of GROUP_M candidate tiles sweep the frame
  // tiles (both operands reused from L2); with on-chip steering only psi is read, so all
  // candidate tiles of one frame tile run together and psi is read from HBM once
  const int gm = GEN ? m_tiles : GROUP_M;
  const int group = tile / (gm * n_tiles);
  const int first_m = group * gm;
  const int gsize = min(m_tiles - first_m, gm);
  const int m_blk = first_m + (tile % (gm * n_tiles)) % gsize;
  const int n_blk = (tile % (gm * n_tiles)) / gsize;
  const int kb_total = (Kd + BLOCK_K - 1) / BLOCK_K;
  const int kper = ((kb_total + ksplit - 1) / ksplit + CHUNK - 1) / CHUNK * CHUNK;
  const int kb0 = ks * kper;                                   // first k-block of this slice
  const int num_kb = max(0, min(kb_total - kb0, kper));        // k-blocks of this slice
  const int num_chunks = (num_kb + CHUNK - 1) / CHUNK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_b);
    if (SPLIT) prefetch_tmap(&map_b2);
    if (!GEN) prefetch_tmap(&map_a);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.full[s], GEN ? 1 + kWorkers : 1);   // TMA + one arrive per generator warp
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.tfull[b], 1);
      mbar_init(&sm.tempty[b], kWorkers);   // one arrive per folding warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  // each role runs to its own exit (no code is shared after the register split):
  // tcgen05 fence + named barrier over the whole CTA, then warp 1 frees TMEM
  auto end_sync = [] {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();                                   // reconverge before the aligned barrier
    asm volatile("bar.sync 1, %0;" ::"n"(kThreadsC) : "memory");
  };
  if (warp < kCtl) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
    if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t kBytes = (BN * SM::NP + (GEN ? 0 : BLOCK_M)) * BLOCK_K * sizeof(float);
      for (int kbl = 0; kbl < num_kb; ++kbl) {
        const int kb = kb0 + kbl;
        const int s = kbl % NS;
        const uint32_t round = kbl / NS;
        mbar_wait(&sm.empty[s], (round & 1) ^ 1);
        mbar_expect_tx(&sm.full[s], kBytes);
        if (!GEN) tma_load_2d(sm.a[s][0], &map_a, &sm.full[s], kb * BLOCK_K, m_blk * BLOCK_M);
        tma_load_2d(sm.b[s][0], &map_b, &sm.full[s], kb * BLOCK_K, n_blk * BN);
        if (SPLIT) tma_load_2d(sm.b[s][SM::NP - 1], &map_b2, &sm.full[s], kb * BLOCK_K, n_blk * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BLOCK_M >> 4) << 24);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int chunk = kb / CHUNK, b = chunk & 1;
        const bool first = (kb % CHUNK) == 0;
        if (first) {   // the fold warps have drained this chunk tile (first two chunks pass)
          mbar_wait(&sm.tempty[b], ((chunk >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const int s = kb % NS;
        const uint32_t round = kb / NS;
        mbar_wait(&sm.full[s], round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = smem_desc(sm.a[s][0]);
        const uint64_t db = smem_desc(sm.b[s][0]);
        const uint64_t da2 = smem_desc(sm.a[s][SM::NP - 1]);
        const uint64_t db2 = smem_desc(sm.b[s][SM::NP - 1]);
        const uint32_t acc = tmem + (uint32_t)(b * BN);
#pragma unroll
        for (int k = 0; k < BLOCK_K / UMMA_K; ++k) {
          const uint64_t off = (uint64_t)((k * UMMA_K * 4) >> 4);
          mma_tf32(acc, da + off, db + off, idesc, (first && k == 0) ? 0u : 1u);
          if (SPLIT) {
            mma_tf32(acc, da + off, db2 + off, idesc, 1);
            mma_tf32(acc, da2 + off, db + off, idesc, 1);
          }
        }
        mma_commit(&sm.empty[s]);
        if ((kb % CHUNK) == CHUNK - 1 || kb == num_kb - 1) mma_commit(&sm.tfull[b]);
      }
    }
    }
    end_sync();
    if (warp == 1) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWorkerRegs));
  {
    const int t = threadIdx.x - 32 * kCtl;     // 0 .. 32 kWorkers - 1
    const int row = t & (BLOCK_M - 1), part = t / BLOCK_M;
    const int64_t gi = (int64_t)m_blk * BLOCK_M + row;
    // fold ownership: TMEM lane quarter (warp % 4) x column slice ((warp - 2) / 4)
    const int quarter = warp & 3, cslice = (warp - kCtl) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    float sum[kFoldCols];
#pragma unroll
    for (int c = 0; c < kFoldCols; ++c) sum[c] = 0.f;
    auto fold = [&](int chunk) {
      const int b = chunk & 1;
      mbar_wait(&sm.tfull[b], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < kFoldCols; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(lane_base + (uint32_t)(b * BN + cslice * kFoldCols + c0), r);
#pragma unroll
        for (int c = 0; c < 32; ++c) sum[c0 + c] += __uint_as_float(r[c]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.tempty[b])) : "memory");
    };
    GenState g;
    gen_state_init(g, kb0 * (BLOCK_K / 2) + kNB * part, gp.B > 0 ? gp.B : 1);
    const int64_t gi_c = gi < J ? gi : J - 1;          // rows past J: any finite values (discarded)
    constexpr uint32_t kPlane = BLOCK_M * BLOCK_K * sizeof(float), kStage = SM::NP * kPlane;
    const uint32_t a_row = smem_u32(&sm.a[0][0][0]) + row * 128;
    const uint32_t full0 = smem_u32(&sm.full[0]), empty0 = smem_u32(&sm.empty[0]);
    uint32_t off[kNB / 2];
#pragma unroll
    for (int qq = 0; qq < kNB / 2; ++qq) off[qq] = (uint32_t)((((kNB / 2) * part + qq) ^ (row & 7)) << 4);
    int folded = 0;
    // two k-blocks per synchronisation round: the generator is latency-bound per round
    // (wait, generate, fence, arrive), so pairing blocks halves the rounds
    static_assert(CHUNK % 2 == 0 && SM::NS % 2 == 0, "k-block pairs must not straddle chunks/rings");
    for (int kb = 0; kb < num_kb; kb += 2) {
      const bool two = kb + 1 < num_kb;
      if (GEN) {
        const int s = kb % NS;
        const uint32_t par = ((kb / NS) & 1) ^ 1;
        mbar_wait_addr(empty0 + 8 * s, par);
        if (two) mbar_wait_addr(empty0 + 8 * (s + 1), par);
        const uint32_t st0 = a_row + s * kStage;
        gen_a_part<SPLIT, kNB>(st0, st0 + (SM::NP - 1) * kPlane, off, (kNB / 2) * part, row & 7, gi_c, gp, g);
        if (two)
          gen_a_part<SPLIT, kNB>(st0 + kStage, st0 + kStage + (SM::NP - 1) * kPlane, off, (kNB / 2) * part,
                                 row & 7, gi_c, gp, g);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // own writes -> async proxy
        __syncwarp();
        if (lane == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * s) : "memory");
          if (two) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * (s + 1)) : "memory");
        }
      }
      if (two && ((kb + 1) % CHUNK) == CHUNK - 1 && (kb + 1) / CHUNK >= 1) fold(folded++);
    }
    while (folded < num_chunks) fold(folded++);
    const int64_t i = (int64_t)m_blk * BLOCK_M + quarter * 32 + lane;
    const bool row_ok = i < J;
    if (zpart) {                                   // split-K: this slice's partial map
#pragma unroll
      for (int c = 0; c < kFoldCols; ++c) {
        const int64_t f = (int64_t)n_blk * BN + cslice * kFoldCols + c;
        if (f >= F) break;
        if (row_ok) zpart[((int64_t)ks * F + f) * J + i] = alpha * sum[c];
      }
      end_sync();
      return;
    }
#pragma unroll
    for (int c = 0; c < kFoldCols; ++c) {
      const int64_t f = (int64_t)n_blk * BN + cslice * kFoldCols + c;
      if (f >= F) break;
      const float v = alpha * sum[c];
      if (z && row_ok) z[f * J + i] = v;
      if (keys) {
        unsigned long long k = row_ok ? make_key(v, (uint32_t)i) : 0ull;
        k = warp_key_max(k);
        if (lane == 0 && k) atomicMax(keys + f, k);
      }
    }
  }
  end_sync();
}

static int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows) {
  return make_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, rows, cols, ld, BLOCK_K, box_rows,
                     "srp_map_tc");
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

// Steering operand straight from the reference's complex128 matrix (srp.py:51-62 /
// an SRPM cache payload, cache.py:1-19): dst[r][2c] = f32(Re H), dst[r][2c+1] = -f32(Im H),
// optionally TF32-rounded (RNE) -- bit-identical to the host conversion conj -> complex64
// -> tf32_rne, so uploads can ship the float64 payload and convert on the GPU.
__global__ void c128_to_steering_kernel(const double2* __restrict__ src, int64_t ld_src, int64_t rows,
                                        int64_t cols, float2* __restrict__ dst, int64_t ld_dst2, int tf32) {
  const int64_t n = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const double2 h = __ldcs(src + r * ld_src + c);
    float re = __double2float_rn(h.x), im = -__double2float_rn(h.y);
    if (tf32) { re = tf32_rne(re); im = tf32_rne(im); }
    dst[r * ld_dst2 + c] = make_float2(re, im);
  }
}

// hi = tf32_rne(x), lo = tf32_rne(x - hi) into two planes (3xTF32 operands)
__global__ void split_tf32_kernel(const float* __restrict__ src, int64_t ld_src, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t ld_dst, int64_t cols) {
  const int64_t r = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ld_dst;
       c += (int64_t)gridDim.x * blockDim.x) {
    float h = 0.f, l = 0.f;
    if (c < cols) {
      const float v = __ldg(src + r * ld_src + c);
      h = tf32_rne(v);
      l = tf32_rne(v - h);
    }
    hi[r * ld_dst + c] = h;
    lo[r * ld_dst + c] = l;
  }
}

// split-K combine: z[f][i] = sum over slices (fixed order) + the per-frame argmax keys
__global__ void splitk_reduce_kernel(const float* __restrict__ zpart, int32_t ksplit, int64_t F, int64_t J,
                                     float* __restrict__ z, unsigned long long* __restrict__ keys) {
  const int64_t f = blockIdx.y;
  unsigned long long best = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < J; i += (int64_t)gridDim.x * blockDim.x) {
    float v = __ldcs(zpart + f * J + i);
#pragma unroll 4
    for (int k = 1; k < ksplit; ++k) v += __ldcs(zpart + ((int64_t)k * F + f) * J + i);
    if (z) __stcs(z + f * J + i, v);
    best = key_max(best, make_key(v, (uint32_t)i));
  }
  if (keys) {
    best = warp_key_max(best);
    if ((threadIdx.x & 31) == 0 && best) atomicMax(keys + f, best);
  }
}

template <bool SPLIT, bool GEN = true>
static int launch_chunked(const float* gcc, int64_t gcc_ld, int64_t F, int32_t Kd, int64_t J, float* z,
                          uint64_t* keys, cudaStream_t st, const GenParams& gp, const float* h2 = nullptr,
                          int64_t h2_ld = 0, int32_t ksplit = 1, float* work = nullptr) {
  CUtensorMap mb, mb2, ma;
  int s = make_map(&mb, gcc, F, Kd, gcc_ld, 256);
  if (s) return s;
  mb2 = mb;
  ma = mb;
  if (SPLIT && (s = make_map(&mb2, gcc + F * gcc_ld, F, Kd, gcc_ld, 256))) return s;
  if (!GEN && (s = make_map(&ma, h2, J, Kd, h2_ld, BLOCK_M))) return s;
  const size_t smem = sizeof(SmemC<SPLIT>) + 1024;
  auto kern = conv_gen_chunked_kernel<SPLIT, GEN>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("srp_map_tdoa: cannot reserve %zu B shared memory", smem);
    return SRPGPU_ERR_LAUNCH;
  }
  const int64_t tiles = ((J + BLOCK_M - 1) / BLOCK_M) * ((F + 255) / 256);
  SRPGPU_CHECK_ARG(tiles < (1ll << 31), SRPGPU_ERR_DIMENSION, "srp_map_tdoa: too many tiles");
  const int kb_total = (Kd + BLOCK_K - 1) / BLOCK_K;
  ksplit = std::max(1, std::min<int32_t>(ksplit, (kb_total + CHUNK - 1) / CHUNK));
  {   // slices hold whole chunks: drop the slices that rounding left empty
    const int kper = ((kb_total + ksplit - 1) / ksplit + CHUNK - 1) / CHUNK * CHUNK;
    ksplit = (kb_total + kper - 1) / kper;
  }
  SRPGPU_CHECK_ARG(ksplit == 1 || work, SRPGPU_ERR_VALUE, "srp_map: split-K needs a work buffer");
  kern<<<(unsigned)(tiles * ksplit), kThreadsC, smem, st>>>(mb, mb2, ma, J, F, Kd, z,
                                                            reinterpret_cast<unsigned long long*>(keys), 2.0f, gp,
                                                            ksplit, ksplit > 1 ? work : nullptr);
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, kern);
      set_error("srp_map_tdoa: launch failed: %s (regs %d, max threads %d, static smem %zu, local %zu, "
                "dynamic smem %zu)", cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock,
                fa.sharedSizeBytes, fa.localSizeBytes, smem);
      return SRPGPU_ERR_LAUNCH;
    }
    count_launch();
  }
  if (ksplit > 1) {
    SRPGPU_CHECK_ARG(F <= 65535, SRPGPU_ERR_DIMENSION, "srp_map: split-K for at most 65535 frames");
    // enough blocks for ~4 per SM, then up to ~8 candidates per thread (one warp key
    // reduction and atomic per several outputs)
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((J + 255) / 256, (4 * num_sms() + F - 1) / F));
    dim3 grid((unsigned)gx, (unsigned)F);
    splitk_reduce_kernel<<<grid, 256, 0, st>>>(work, ksplit, F, J, z, reinterpret_cast<unsigned long long*>(keys));
    SRPGPU_CHECK_LAUNCH("srp_map(split-K reduce)");
  }
  return SRPGPU_OK;
}

}  // namespace tc

int reset_keys(uint64_t* keys, int64_t F, cudaStream_t st);

}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_c128_to_steering(const void* src, int64_t ld_src, int64_t rows, int64_t cols, float* dst,
                                       int64_t ld_dst, int32_t tf32, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(rows >= 0 && cols >= 0 && ld_src >= cols && ld_dst >= 2 * cols && ld_dst % 2 == 0,
                   SRPGPU_ERR_DIMENSION, "c128_to_steering: bad pitches");
  SRPGPU_CHECK_ARG(((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 7) == 0, SRPGPU_ERR_VALUE,
                   "c128_to_steering: misaligned operands");
  if (rows == 0 || cols == 0) return SRPGPU_OK;
  const int64_t n = rows * cols;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 16 * (int64_t)num_sms());
  tc::c128_to_steering_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const double2*>(src), ld_src, rows, cols, reinterpret_cast<float2*>(dst), ld_dst / 2, tf32);
  SRPGPU_CHECK_LAUNCH("c128_to_steering");
  return SRPGPU_OK;
}

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

extern "C" int srpgpu_split_tf32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int64_t rows,
                                 int64_t cols, srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(ld_dst >= cols && ld_src >= cols && rows >= 0, SRPGPU_ERR_DIMENSION,
                   "split_tf32: bad pitches");
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>((ld_dst + 255) / 256, 64), (unsigned)nr);
    tc::split_tf32_kernel<<<grid, 256, 0, as_stream(stream)>>>(src + r0 * ld_src, ld_src, dst + r0 * ld_dst,
                                                                dst + (rows + r0) * ld_dst, ld_dst, cols);
    SRPGPU_CHECK_LAUNCH("split_tf32");
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_srp_map_tc(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t gcc_len,
                                 const float* h2, int64_t h2_ld, int64_t num_candidates, int32_t ksplit,
                                 float* work, float* z, uint64_t* keys, srpgpu_stream_t stream) {
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
  (void)m_tiles; (void)n256;
  // chunked TMEM accumulation folded into fp32 registers (see conv_gen_chunked_kernel)
  return tc::launch_chunked<false, false>(gcc, gcc_ld, num_frames, Kd, num_candidates, z, keys, st, gp, h2,
                                          h2_ld, ksplit, work);
}

extern "C" int srpgpu_srp_map_tdoa(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t num_pairs,
                                   int32_t half_len, const float* xtab, int64_t num_candidates,
                                   int32_t split, int32_t ksplit, float* work, float* z, uint64_t* keys,
                                   srpgpu_stream_t stream) {
  const int32_t bins = half_len - 1;
  const int32_t Kd = 2 * num_pairs * bins;
  SRPGPU_CHECK_ARG(num_pairs >= 1 && bins >= 1 && num_candidates >= 1, SRPGPU_ERR_DIMENSION,
                   "srp_map_tdoa: empty operator");
  SRPGPU_CHECK_ARG(bins >= 16, SRPGPU_ERR_UNSUPPORTED, "srp_map_tdoa: frames shorter than 34 samples");
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
  (void)m_tiles; (void)n256;
  // chunked TMEM accumulation folded into fp32 registers (bounded in-pipe accumulation)
  if (split)   // 3xTF32: gcc holds the hi plane [F][gcc_ld] followed by the lo plane
    return tc::launch_chunked<true>(gcc, gcc_ld, num_frames, Kd, num_candidates, z, keys, st, gp, nullptr, 0,
                                    ksplit, work);
  return tc::launch_chunked<false>(gcc, gcc_ld, num_frames, Kd, num_candidates, z, keys, st, gp, nullptr, 0,
                                   ksplit, work);
}
