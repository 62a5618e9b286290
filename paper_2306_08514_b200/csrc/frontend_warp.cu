// Warp-per-frame frontend for frame lengths L = 32 * LP (LP = 8, 16, 32: L = 256, 512, 1024).
//
// Same math as frontend.cu (frontend.py:89-160, sampling.py:106-134), laid out for
// sm_100a: every warp owns one frame at a time and never waits on other warps.
//   * FFT of length L = 32 x LP by the four-step method: each lane holds 32
//     points in registers and runs a 32-point radix-2 DIF transform with
//     compile-time twiddles; the W_L^{l k2} twiddles come from a CTA table laid
//     out [k2][l] (conflict-free); one padded shared-memory transpose; then
//     32/LP transforms of LP points per lane.  A warp runs 32/LP FFTs at once.
//   * two real channels are packed into one complex FFT (forward) and two
//     pairs' Hermitian spectra into one complex FFT (inverse, as conj(FFT(conj))).
//   * the inverse is pruned: only the 2N_p+1 kept lags (|n| <= N_p) are produced,
//     i.e. outputs k1 in {0, LP-1} of the second step when N_p < 32.
//   * frame energy for the PHAT floor by warp shuffles.
#include <cstdlib>
#include <cuda_bf16.h>

#include "frontend_warp.cuh"

namespace srpgpu {

namespace wf {

// W_32^m = exp(-2 pi i m / 32) for m in [0, 16); folded to immediates after unrolling
__device__ __forceinline__ float2 w32(int m) {
  switch (m & 15) {
    case 0: return make_float2(1.0f, 0.0f);
    case 1: return make_float2(0.98078528040323043f, -0.19509032201612825f);
    case 2: return make_float2(0.92387953251128674f, -0.38268343236508978f);
    case 3: return make_float2(0.83146961230254524f, -0.55557023301960218f);
    case 4: return make_float2(0.70710678118654752f, -0.70710678118654752f);
    case 5: return make_float2(0.55557023301960218f, -0.83146961230254524f);
    case 6: return make_float2(0.38268343236508978f, -0.92387953251128674f);
    case 7: return make_float2(0.19509032201612825f, -0.98078528040323043f);
    case 8: return make_float2(0.0f, -1.0f);
    case 9: return make_float2(-0.19509032201612825f, -0.98078528040323043f);
    case 10: return make_float2(-0.38268343236508978f, -0.92387953251128674f);
    case 11: return make_float2(-0.55557023301960218f, -0.83146961230254524f);
    case 12: return make_float2(-0.70710678118654752f, -0.70710678118654752f);
    case 13: return make_float2(-0.83146961230254524f, -0.55557023301960218f);
    case 14: return make_float2(-0.92387953251128674f, -0.38268343236508978f);
    default: return make_float2(-0.98078528040323043f, -0.19509032201612825f);
  }
}

__device__ __forceinline__ float2 twmul32(float2 d, int m) {  // d * W_32^m, m in [0, 16)
  if (m == 0) return d;
  if (m == 8) return make_float2(d.y, -d.x);
  const float2 w = w32(m);
  return make_float2(d.x * w.x - d.y * w.y, d.x * w.y + d.y * w.x);
}

// in-place radix-2 DIF over v[base .. base+N) in registers (base constant after unrolling):
// natural order in, v[base + i] = X[bitrev(i)] out
template <int N>
__device__ __forceinline__ void dif(float2 (&v)[32], const int base) {
#pragma unroll
  for (int h = N / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int b = 0; b < N; b += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 a = v[base + b + j], c = v[base + b + j + h];
        v[base + b + j] = make_float2(a.x + c.x, a.y + c.y);
        v[base + b + j + h] = twmul32(make_float2(a.x - c.x, a.y - c.y), j * (32 / (2 * h)));
      }
    }
  }
}

template <int N>
__host__ __device__ constexpr int brev(int i) {
  int r = 0;
  for (int b = 1, o = N >> 1; b < N; b <<= 1, o >>= 1)
    if (i & b) r |= o;
  return r;
}

template <int LP>
struct Geo {
  static constexpr int L = 32 * LP;
  static constexpr int K = L / 2;
  static constexpr int R = 32 / LP;            // FFTs per warp
  static constexpr int XP = 32 * (LP + 1);     // float2 per FFT transpose area (padded)
  static constexpr int WORK = R * XP;          // float2 per warp work area
};

// Forward FFT of the 32 points v[j] = x[fl + LP*j] of this lane's FFT.
// On return v[r*LP + i] = X[32*brev_LP(i) + fl + LP*r]  (FULL2), or only the
// k1 in {0, LP-1} outputs in v[r*LP + 0] and v[r*LP + 1] (pruned).
template <int LP, bool FULL2>
__device__ __forceinline__ void fft_l(float2 (&v)[32], float2* xp, const float2* twT, int fl) {
  dif<32>(v, 0);                                // v[i] = A[brev5(i)]
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int k2 = brev<32>(i);
    v[i] = cmul(v[i], twT[k2 * LP + fl]);       // W_L^{fl k2}
    xp[k2 * (LP + 1) + fl] = v[i];
  }
  __syncwarp();
  constexpr int R = 32 / LP;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float2* row = xp + (fl + LP * r) * (LP + 1);
#pragma unroll
    for (int n1 = 0; n1 < LP; ++n1) v[r * LP + n1] = row[n1];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (FULL2) {
      dif<LP>(v, r * LP);
    } else {
      // X[0] = sum u ; X[LP-1] = sum u W_LP^{-n1} = sum u conj(W_32^{n1*32/LP})
      float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int n1 = 0; n1 < LP; ++n1) {
        const float2 u = v[r * LP + n1];
        s0.x += u.x;
        s0.y += u.y;
        const int m = (n1 * (32 / LP)) & 31;
        float2 w = (m < 16) ? w32(m) : make_float2(-w32(m - 16).x, -w32(m - 16).y);
        w.y = -w.y;   // conj
        s1.x += u.x * w.x - u.y * w.y;
        s1.y += u.x * w.y + u.y * w.x;
      }
      v[r * LP + 0] = s0;
      v[r * LP + 1] = s1;
    }
  }
}

__device__ __forceinline__ float2 cross_phat(const float2* spec, int Kp1, int m, int mp, int k, const Phat& ph) {
  const float2 a = spec[m * Kp1 + k];
  const float2 b = spec[mp * Kp1 + k];
  return ph(cmulc(a, b));
}

// forward FFTs of one frame (R channel pairs per round, rounds split over the frame's warps)
// into the shared spectra [M][K+1]; returns this warp's share of sum |Y|^2
template <int LP, int kWpf>
__device__ __forceinline__ float forward_frame(const WarpParams& prm, int64_t start, float2* spec, float2* work,
                                               float2* xp, const float2* twT, int lane, int mi) {
  using G = Geo<LP>;
  constexpr int L = G::L, K = G::K, R = G::R, Kp1 = K + 1;
  const int M = prm.M;
  const int fi = lane / LP, fl = lane % LP;
  float energy = 0.f;
  // ---------------- forward FFTs: R channel pairs per round, rounds split over the warps ----
  for (int c0 = 2 * R * mi; c0 < M; c0 += 2 * R * kWpf) {
    const int ca = c0 + 2 * fi, cb = ca + 1;
    float2 v[32];
    const float* xa = prm.samples + (int64_t)ca * prm.ld_samples + start;
    const float* xb = prm.samples + (int64_t)cb * prm.ld_samples + start;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = fl + LP * j;
      const float w = __ldg(prm.window + n);
      const float a = (ca < M) ? __ldg(xa + n) * w : 0.f;
      const float b = (cb < M) ? __ldg(xb + n) * w : 0.f;
      v[j] = make_float2(a, b);
    }
    fft_l<LP, true>(v, xp, twT, fl);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < LP; ++i) xp[32 * brev<LP>(i) + fl + LP * r] = v[r * LP + i];
    __syncwarp();
    // unpack the two real spectra: Ya = (Z + conj Z[L-k]) / 2, Yb = (Z - conj Z[L-k]) / 2j
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int qa = c0 + 2 * q, qb = qa + 1;
      if (qa >= M) break;
      const float2* zq = work + q * G::XP;
      for (int k = lane; k < Kp1; k += 32) {
        const float2 Z = zq[k];
        const float2 Zc = conjf2(zq[(L - k) & (L - 1)]);
        const float2 Ya = make_float2(0.5f * (Z.x + Zc.x), 0.5f * (Z.y + Zc.y));
        spec[qa * Kp1 + k] = Ya;
        energy += Ya.x * Ya.x + Ya.y * Ya.y;
        if (qb < M) {
          const float2 Yb = make_float2(0.5f * (Z.y - Zc.y), -0.5f * (Z.x - Zc.x));
          spec[qb * Kp1 + k] = Yb;
          energy += Yb.x * Yb.x + Yb.y * Yb.y;
        }
      }
    }
    __syncwarp();
  }
  return energy;
}

// PHAT cross-spectra + pruned inverse FFTs of one frame's pairs (two pairs per FFT, rounds
// split over the frame's warps); every kept lag goes to put(offset, N_p, storage index, value)
template <int LP, int kWpf, class Put>
__device__ __forceinline__ void inverse_frame(const WarpParams& prm, const float2* spec, float2* work, float2* xp,
                                              const float2* twT, const int* s_pairs, const int* s_counts,
                                              const int* s_off, const Phat& ph, int lane, int mi, const Put& put) {
  using G = Geo<LP>;
  constexpr int L = G::L, K = G::K, R = G::R, Kp1 = K + 1, B = K - 1;
  const int P = prm.P;
  const int fi = lane / LP, fl = lane % LP;
  for (int p0 = 2 * R * mi; p0 < P; p0 += 2 * R * kWpf) {
    // PHAT cross-spectra of this round's pairs into each FFT's work area: [2][B]
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int pa = p0 + 2 * q, pb = pa + 1;
      if (pa >= P) break;
      float2* sq = work + q * G::XP;
      const int ma = s_pairs[2 * pa], mpa = s_pairs[2 * pa + 1];
      const int mb = (pb < P) ? s_pairs[2 * pb] : 0, mpb = (pb < P) ? s_pairs[2 * pb + 1] : 0;
      for (int k = 1 + lane; k < K; k += 32) {
        sq[k - 1] = cross_phat(spec, Kp1, ma, mpa, k, ph);
        sq[B + k - 1] = (pb < P) ? cross_phat(spec, Kp1, mb, mpb, k, ph)
                                 : make_float2(0.f, 0.f);
      }
    }
    __syncwarp();
    const int pa = p0 + 2 * fi, pb = pa + 1;
    float2 v[32];
    {
      const float2* sa = xp;
      const float2* sb = xp + B;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int k = fl + LP * j;
        float2 z = make_float2(0.f, 0.f);
        if (pa < P && k != 0 && k != K) {
          if (k < K) {
            const float2 a = sa[k - 1], c = sb[k - 1];
            z = make_float2(a.x - c.y, a.y + c.x);      // a + j c
          } else {
            const float2 a = sa[L - k - 1], c = sb[L - k - 1];
            z = make_float2(a.x + c.y, -a.y + c.x);     // conj(a) + j conj(c)
          }
        }
        v[j] = conjf2(z);
      }
    }
    __syncwarp();
    // prune the second FFT step when every kept lag of the warp's pairs has |n| < 32
    int nmax = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int qa = p0 + 2 * q;
      if (qa < P) nmax = max(nmax, s_counts[qa]);
      if (qa + 1 < P) nmax = max(nmax, s_counts[qa + 1]);
    }
    const bool full2 = nmax >= 32;
    if (full2) fft_l<LP, true>(v, xp, twT, fl);
    else fft_l<LP, false>(v, xp, twT, fl);
    if (pa < P) {
      const int Na = s_counts[pa], oa = s_off[pa];
      const int Nb = (pb < P) ? s_counts[pb] : -1, ob = (pb < P) ? s_off[pb] : 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k2 = fl + LP * r;
        if (full2) {
#pragma unroll
          for (int i = 0; i < LP; ++i) {
            const int n = 32 * brev<LP>(i) + k2;
            const float2 x = v[r * LP + i];
            const int da = (n <= Na) ? n : ((L - n <= Na) ? 2 * Na + 1 - (L - n) : -1);
            if (da >= 0) put(oa, Na, da, x.x);
            const int db = (n <= Nb) ? n : ((L - n <= Nb) ? 2 * Nb + 1 - (L - n) : -1);
            if (db >= 0) put(ob, Nb, db, -x.y);
          }
        } else {
          const float2 x0 = v[r * LP + 0];   // n = k2
          const float2 x1 = v[r * LP + 1];   // n = L - 32 + k2, distance d = 32 - k2
          const int d = 32 - k2;
          if (k2 <= Na) put(oa, Na, k2, x0.x);
          if (d <= Na) put(oa, Na, 2 * Na + 1 - d, x1.x);
          if (k2 <= Nb) put(ob, Nb, k2, -x0.y);
          if (d <= Nb) put(ob, Nb, 2 * Nb + 1 - d, -x1.y);
        }
      }
    }
    __syncwarp();
  }
}

// xi sink of the unfused chain: global f32 samples (+ bf16 planes)
struct GlobalXi {
  const WarpParams& prm;
  float* dst;
  int64_t sst;
  int64_t f;
  __device__ __forceinline__ void operator()(int o, int N, int d, float v) const { put_xi(prm, dst, sst, f, o, N, d, v); }
};

constexpr int kWarps = 4;   // per CTA

// named barrier of the kWpf warps sharing one frame (kWpf == 1: the warp itself)
template <int kWpf>
__device__ __forceinline__ void frame_sync(int fg) {
  if (kWpf == 1) {
    __syncwarp();
  } else if (kWpf == 2) {
    if (fg == 0) asm volatile("bar.sync 1, 64;" ::: "memory");
    else asm volatile("bar.sync 2, 64;" ::: "memory");
  } else {
    __syncthreads();
  }
}

// kWpf warps per frame share its spectra: 1 (latency-bound small batches: a warp per
// frame) or 2 (large batches: half the spectra buffers per warp -> more resident warps)
// register budget: 4 CTAs per SM (<= 128 registers, no spills; left free the compiler takes
// up to ~250 and only 2 CTAs fit) -- cfg3, 10^4 frames: 0.37 vs 0.47 ms; 10^4 cfg2-shaped
// frames: 0.20 vs 0.24 ms.  The 1-warp-per-frame L = 1024 kernel of small batches keeps the
// free allocation (a few % faster at 1000 frames).  -DWARP_MINB_ALL=n overrides (A/B builds).
template <int LP, int kWpf>
struct WarpMinBlocks {
#ifdef WARP_MINB_ALL
  static constexpr int value = WARP_MINB_ALL;
#else
  static constexpr int value = (LP == 32 && kWpf == 1) ? 1 : 4;
#endif
};

template <int LP, int OUT, int kWpf>
__global__ void __launch_bounds__(kWarps * 32, WarpMinBlocks<LP, kWpf>::value)
frontend_warp_kernel(const WarpParams prm) {
  using G = Geo<LP>;
  constexpr int L = G::L, K = G::K, R = G::R;
  constexpr int Kp1 = K + 1, B = K - 1;
  constexpr int kFpc = kWarps / kWpf;                                   // frames per CTA
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* twT = reinterpret_cast<float2*>(smem_raw);                    // [32][LP]
  int* s_pairs = reinterpret_cast<int*>(twT + 32 * LP);                 // [2P]
  int* s_counts = s_pairs + 2 * prm.P;                                  // [P]
  int* s_off = s_counts + prm.P;                                        // [P+1]
  float* s_energy = reinterpret_cast<float*>(s_off + prm.P + 1);        // [kWarps]
  const size_t head = (((size_t)32 * LP * 8 + (size_t)(4 * prm.P + 1 + kWarps) * 4) + 15) & ~(size_t)15;
  const int M = prm.M, P = prm.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int fg = wid / kWpf, mi = wid % kWpf;
  const size_t frame_bytes = ((size_t)M * Kp1 + kWpf * G::WORK) * sizeof(float2);
  float2* spec = reinterpret_cast<float2*>(smem_raw + head + fg * frame_bytes);   // [M][K+1], shared
  float2* work = spec + (size_t)M * Kp1 + mi * G::WORK;                           // [R][XP], per warp
  const int fi = lane / LP, fl = lane % LP;
  float2* xp = work + fi * G::XP;

  for (int e = threadIdx.x; e < 32 * LP; e += blockDim.x) {
    const int k2 = e / LP, l = e % LP;
    float sn, cs;
    sincospif(2.0f * (float)(k2 * l) / (float)L, &sn, &cs);
    twT[e] = make_float2(cs, -sn);
  }
  for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) s_pairs[i] = prm.pairs[i];
  if (OUT == W_OUT_XI) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_counts[i] = prm.counts[i];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) s_off[i] = prm.offsets[i];
  }
  __syncthreads();

  const int64_t total_groups = (int64_t)gridDim.x * kFpc;
  for (int64_t f = (int64_t)blockIdx.x * kFpc + fg; f < prm.F; f += total_groups) {
    const int64_t start = (prm.first_frame + f) * (int64_t)prm.hop;
    float energy = forward_frame<LP, kWpf>(prm, start, spec, work, xp, twT, lane, mi);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
    if (lane == 0) s_energy[wid] = energy;
    frame_sync<kWpf>(fg);                            // spectra + energy of the frame complete
    float floor = prm.floor_value;
    if (prm.weighting && prm.floor_mode == 0) {
      float e = 0.f;
#pragma unroll
      for (int w = 0; w < kWpf; ++w) e += s_energy[fg * kWpf + w];
      floor = prm.floor_value * e;
    }
    const Phat ph(prm.weighting, floor);

    if (OUT == W_OUT_GCC) {
      float2* dst = prm.gcc_out + f * prm.gcc_ld;
      for (int p = mi; p < P; p += kWpf) {
        const int m = s_pairs[2 * p], mp = s_pairs[2 * p + 1];
        for (int k = 1 + lane; k < K; k += 32) {
          float2 val = cross_phat(spec, Kp1, m, mp, k, ph);
          if (prm.round_tf32) val = make_float2(tf32_rne(val.x), tf32_rne(val.y));
          dst[p * B + k - 1] = val;
        }
      }
      for (int64_t idx = (int64_t)P * B + lane + 32 * mi; idx < prm.gcc_ld; idx += 32 * kWpf)
        dst[idx] = make_float2(0.f, 0.f);
    } else {
      float* dst = prm.xi_out + (prm.xi_ld ? f : f * (int64_t)prm.S);
      const int64_t sst = prm.xi_ld ? prm.xi_ld : 1;
      inverse_frame<LP, kWpf>(prm, spec, work, xp, twT, s_pairs, s_counts, s_off, ph, lane, mi,
                              GlobalXi{prm, dst, sst, f});
      if (prm.xi_planes && !prm.planes_ld && mi == 0) {   // zero the planes' pad columns [S, cols8)
        uint16_t* pl = prm.xi_planes + f * prm.cols8;
        for (int c = prm.S + lane; c < prm.cols8; c += 32) {
          pl[c] = 0;
          pl[prm.F * prm.cols8 + c] = 0;
        }
      }
    }
    frame_sync<kWpf>(fg);                            // spectra free for the next frame
  }
}

struct SmemXi {
  float* xs;
  int fg;
  __device__ __forceinline__ void operator()(int o, int, int d, float v) const { xs[(o + d) * 4 + fg] = v; }
};

constexpr int kMapW = 16;   // operator entries per chunk taken by the unrolled (all loads first) path

// running per-lane argmax of the CTA's 4 frames: ordered float bits (the packed-key order:
// largest value, NaN above everything, -0 == +0) and the first candidate reaching it
struct Best4 {
  uint32_t ob[4];
  int32_t idx[4];
  __device__ __forceinline__ Best4() {
#pragma unroll
    for (int fr = 0; fr < 4; ++fr) {
      ob[fr] = 0u;
      idx[fr] = -1;
    }
  }
  __device__ __forceinline__ unsigned long long key(int fr) const {
    return idx[fr] < 0 ? 0ull : ((unsigned long long)ob[fr] << 32) | (0xFFFFFFFFull - (uint32_t)idx[fr]);
  }
};

// one candidate's map values for the CTA's 4 frames: z stores + running argmax (a lane's
// candidates arrive in increasing index order, so strict '>' keeps the first maximum)
__device__ __forceinline__ void emit4(float4 acc, int64_t i, int64_t J, int64_t fbase, int nvalid, float* z,
                                      Best4& best) {
  if (i >= J) return;
  const float a[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
  for (int fr = 0; fr < 4; ++fr) {
    if (z && fr < nvalid) __stcs(z + (fbase + fr) * J + i, a[fr]);
    const uint32_t ob = ordered_bits(a[fr]);
    if (best.idx[fr] < 0 || ob > best.ob[fr]) {
      best.ob[fr] = ob;
      best.idx[fr] = (int32_t)i;
    }
  }
}

__device__ __forceinline__ void fma4(float4& acc, float w, float4 x) {
  acc.x = fmaf(w, x.x, acc.x);
  acc.y = fmaf(w, x.y, acc.y);
  acc.z = fmaf(w, x.z, acc.z);
  acc.w = fmaf(w, x.w, acc.w);
}

// SSPI map phase: sliced-ELL sparse operator (interpolation.py:188-195)
struct SellPhase {
  SellMap mp;
  static size_t smem(const SellMap& m, int) { return (size_t)((m.J + 31) / 32 + 1) * 4; }
  __device__ __forceinline__ const SellMap& out() const { return mp; }
  __device__ __forceinline__ void setup(void* extra) const {
    int* s_choff = reinterpret_cast<int*>(extra);
    const int nch = (int)((mp.J + 31) / 32);
    for (int i = threadIdx.x; i <= nch; i += blockDim.x) s_choff[i] = mp.chunk_off[i];
  }
  __device__ __forceinline__ void prepare(const float4*, void*, int, int) const {}
  __device__ __forceinline__ void candidates(const float4* xs4, const void* extra, int64_t fbase, int nvalid,
                                             int wid, int lane, Best4& best) const {
    const int* s_choff = reinterpret_cast<const int*>(extra);
    const int64_t J = mp.J;
    const int nch = (int)((J + 31) / 32);
    // two chunks per warp at a time, all their entries loaded before any is used (the
    // operator streams from L2: issue every load of both chunks, then do the FMAs)
    for (int c = wid; c < nch; c += 2 * kWarps) {
      const int cb = c + kWarps;
      const int ea = s_choff[c], na = s_choff[c + 1] - ea;
      const int eb = cb < nch ? s_choff[cb] : 0, nb = cb < nch ? s_choff[cb + 1] - eb : 0;
      float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
      const bool has_b = cb < nch;
      if (na == kMapW && (!has_b || nb == kMapW)) {
        // chunks padded to kMapW entries on the host: unconditional loads at fixed offsets
        const uint16_t* ca = mp.cols + (int64_t)ea * 32 + lane;
        const float* va = mp.vals + (int64_t)ea * 32 + lane;
        const uint16_t* cbp = mp.cols + (int64_t)eb * 32 + lane;
        const float* vb = mp.vals + (int64_t)eb * 32 + lane;
        uint32_t col[2][kMapW];
        float wv[2][kMapW];
#pragma unroll
        for (int t = 0; t < kMapW; ++t) {
          col[0][t] = __ldg(ca + t * 32);
          wv[0][t] = __ldg(va + t * 32);
        }
        if (has_b) {
#pragma unroll
          for (int t = 0; t < kMapW; ++t) {
            col[1][t] = __ldg(cbp + t * 32);
            wv[1][t] = __ldg(vb + t * 32);
          }
        }
#pragma unroll
        for (int t = 0; t < kMapW; ++t) fma4(acc[0], wv[0][t], xs4[col[0][t]]);
        if (has_b) {
#pragma unroll
          for (int t = 0; t < kMapW; ++t) fma4(acc[1], wv[1][t], xs4[col[1][t]]);
        }
      } else {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int e0 = h ? eb : ea, n = h ? nb : na;
          if (n == 2 * kMapW) {        // chunks padded to 32 entries: one chunk, all loads first
            const uint16_t* cp = mp.cols + (int64_t)e0 * 32 + lane;
            const float* vp = mp.vals + (int64_t)e0 * 32 + lane;
            uint32_t col[2 * kMapW];
            float wv[2 * kMapW];
#pragma unroll
            for (int t = 0; t < 2 * kMapW; ++t) {
              col[t] = __ldg(cp + t * 32);
              wv[t] = __ldg(vp + t * 32);
            }
#pragma unroll
            for (int t = 0; t < 2 * kMapW; ++t) fma4(acc[h], wv[t], xs4[col[t]]);
          } else {
#pragma unroll 4
            for (int e = e0; e < e0 + n; ++e)
              fma4(acc[h], __ldg(mp.vals + (int64_t)e * 32 + lane), xs4[__ldg(mp.cols + (int64_t)e * 32 + lane)]);
          }
        }
      }
      emit4(acc[0], (int64_t)c * 32 + lane, J, fbase, nvalid, mp.z, best);
      emit4(acc[1], (int64_t)cb * 32 + lane, J, fbase, nvalid, mp.z, best);
    }
  }
};

// SLRI map phase: z = tall (fat xi) (interpolation.py:178-185); y [R][4 frames] in shared memory
struct SlriPhase {
  SlriMap mp;
  static size_t smem(const SlriMap& m, int) { return (size_t)((m.R + 15) / 16 * 16) * 16; }
  __device__ __forceinline__ const SlriMap& out() const { return mp; }
  __device__ __forceinline__ void setup(void*) const {}
  __device__ __forceinline__ void prepare(const float4* xs4, void* extra, int wid, int lane) const {
    float4* ys = reinterpret_cast<float4*>(extra);
    for (int r = mp.R + threadIdx.x; r < (mp.R + 15) / 16 * 16; r += blockDim.x)
      ys[r] = make_float4(0.f, 0.f, 0.f, 0.f);       // padding rows of tall_t are zero too
    for (int r = wid; r < mp.R; r += kWarps) {        // y[r] = fat[r] . xi for the 4 frames
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      const float* fr = mp.fat + (int64_t)r * mp.S;
      for (int s = lane; s < mp.S; s += 32) fma4(acc, __ldg(fr + s), xs4[s]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
      }
      if (lane == 0) ys[r] = acc;
    }
  }
  __device__ __forceinline__ void candidates(const float4*, const void* extra, int64_t fbase, int nvalid, int wid,
                                             int lane, Best4& best) const {
    const float4* ys = reinterpret_cast<const float4*>(extra);
    const int64_t J = mp.J;
    const int nch = (int)((J + 31) / 32);
    // two 32-candidate chunks per warp at a time; tall_t has R rounded up to 16 rows (zero
    // padded on the host), loaded 16 rows x 2 chunks before any FMA
    for (int c = wid; c < nch; c += 2 * kWarps) {
      const int cb = c + kWarps;
      const bool has_b = cb < nch;
      const int64_t ia = (int64_t)c * 32 + lane, ib = (int64_t)cb * 32 + lane;
      const float* ta = mp.tallT + (ia < J ? ia : 0);
      const float* tb = mp.tallT + (has_b && ib < J ? ib : 0);
      float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
      for (int r0 = 0; r0 < mp.R; r0 += 16) {
        float t[2][16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[0][u] = __ldg(ta + (int64_t)(r0 + u) * J);
        if (has_b) {
#pragma unroll
          for (int u = 0; u < 16; ++u) t[1][u] = __ldg(tb + (int64_t)(r0 + u) * J);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) fma4(acc[0], t[0][u], ys[r0 + u]);
        if (has_b) {
#pragma unroll
          for (int u = 0; u < 16; ++u) fma4(acc[1], t[1][u], ys[r0 + u]);
        }
      }
      emit4(acc[0], ia, J, fbase, nvalid, mp.z, best);
      if (has_b) emit4(acc[1], ib, J, fbase, nvalid, mp.z, best);
    }
  }
};

// Fused chain for latency-scale batches: samples -> spectra -> PHAT ->
// pruned inverse FFT -> map -> per-frame argmax in ONE kernel.  A CTA's 4 warps each run
// one frame's frontend (the warp-per-frame code above) with the TD-GCC samples kept in
// shared memory as xs[S][4] (frame fastest); then the 4 warps evaluate the map for all 4
// frames at once (one float4 shared load feeds 4 FMAs): the SSPI sliced-ELL operator or
// the SLRI factors, read coalesced through L1 / L2.  z is written once; one CTA owns its
// frames, so the argmax index is written directly (no key reset, no atomics, no decode).
// kWpf warps per frame: 1 (4 frames per CTA: the map phase reuses each operator load for 4
// frames) or 4 (1 frame per CTA for tiny batches: the frame's FFT rounds run side by side)
template <int LP, class Phase, int kWpf>
__global__ void __launch_bounds__(kWarps * 32)
frontend_map_kernel(const WarpParams prm, const Phase ph) {
  using G = Geo<LP>;
  constexpr int L = G::L, K = G::K;
  constexpr int Kp1 = K + 1;
  constexpr int kFpc = kWarps / kWpf;                                   // frames per CTA
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* twT = reinterpret_cast<float2*>(smem_raw);                    // [32][LP]
  int* s_pairs = reinterpret_cast<int*>(twT + 32 * LP);                 // [2P]
  int* s_counts = s_pairs + 2 * prm.P;                                  // [P]
  int* s_off = s_counts + prm.P;                                        // [P+1]
  const size_t head = (((size_t)32 * LP * 8 + (size_t)(4 * prm.P + 1) * 4) + 15) & ~(size_t)15;
  const int M = prm.M, P = prm.P, S = prm.S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int fg = wid / kWpf, mi = wid % kWpf;
  const size_t frame_bytes = ((size_t)M * Kp1 + kWpf * G::WORK) * sizeof(float2);
  float2* spec = reinterpret_cast<float2*>(smem_raw + head + fg * frame_bytes);   // [M][K+1]
  float2* work = spec + (size_t)M * Kp1 + mi * G::WORK;                           // [R][XP]
  float* xs = reinterpret_cast<float*>(smem_raw + head + kFpc * frame_bytes);     // [S][4]
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(xs + 4 * (size_t)S);   // [4 warps][4]
  float* s_energy = reinterpret_cast<float*>(s_keys + 16);                                  // [4 warps]
  void* extra = s_energy + kWarps;                                                          // phase data
  float2* xp = work + (lane / LP) * G::XP;

  for (int e = threadIdx.x; e < 32 * LP; e += blockDim.x) {
    const int k2 = e / LP, l = e % LP;
    float sn, cs;
    sincospif(2.0f * (float)(k2 * l) / (float)L, &sn, &cs);
    twT[e] = make_float2(cs, -sn);
  }
  for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) s_pairs[i] = prm.pairs[i];
  for (int i = threadIdx.x; i < P; i += blockDim.x) s_counts[i] = prm.counts[i];
  for (int i = threadIdx.x; i <= P; i += blockDim.x) s_off[i] = prm.offsets[i];
  if (kFpc < 4)                                       // columns no frame writes stay zero
    for (int i = threadIdx.x; i < 4 * S; i += blockDim.x) xs[i] = 0.f;
  ph.setup(extra);
  __syncthreads();

  const float4* xs4 = reinterpret_cast<const float4*>(xs);
  const int64_t groups = (prm.F + kFpc - 1) / kFpc;
  const auto& out = ph.out();
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const int64_t fbase = g * kFpc;
    const int64_t left = prm.F - fbase;
    const int nvalid = left < kFpc ? (int)left : kFpc;
    const int64_t f = fbase + fg;
    if (fg < nvalid) {                                // warp-uniform per frame group
      const int64_t start = (prm.first_frame + f) * (int64_t)prm.hop;
      float energy = forward_frame<LP, kWpf>(prm, start, spec, work, xp, twT, lane, mi);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
      if (kWpf > 1) {
        if (lane == 0) s_energy[wid] = energy;
        frame_sync<kWpf>(fg);                         // spectra + energy of the frame complete
        energy = 0.f;
#pragma unroll
        for (int w = 0; w < kWpf; ++w) energy += s_energy[fg * kWpf + w];
      }
      const float floor = (prm.weighting && prm.floor_mode == 0) ? prm.floor_value * energy : prm.floor_value;
      inverse_frame<LP, kWpf>(prm, spec, work, xp, twT, s_pairs, s_counts, s_off, Phat(prm.weighting, floor), lane,
                              mi, SmemXi{xs, fg});
    } else if (mi == 0) {
      for (int s = lane; s < S; s += 32) xs[s * 4 + fg] = 0.f;
    }
    __syncthreads();                                  // xs of the CTA's frames complete
    ph.prepare(xs4, extra, wid, lane);
    __syncthreads();
    Best4 lane_best;
    ph.candidates(xs4, extra, fbase, nvalid, wid, lane, lane_best);
    unsigned long long best[4];
#pragma unroll
    for (int fr = 0; fr < 4; ++fr) best[fr] = warp_key_max(lane_best.key(fr));
    if (lane == 0) {
#pragma unroll
      for (int fr = 0; fr < 4; ++fr) s_keys[wid * 4 + fr] = best[fr];
    }
    __syncthreads();                                  // xs free; s_keys complete
    if (wid == 0 && lane < nvalid) {
      unsigned long long k = s_keys[lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) k = key_max(k, s_keys[w * 4 + lane]);
      if (out.keys) out.keys[fbase + lane] = k;
      if (out.index) out.index[fbase + lane] = (int64_t)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
    }
  }
}

template <int LP, class Phase, int kWpf, class Map>
static int launch_fused_w(const WarpParams& wp, const Map& mp, cudaStream_t st, const char* what) {
  using G = Geo<LP>;
  constexpr int kFpc = kWarps / kWpf;
  const size_t head = (((size_t)32 * LP * 8 + (size_t)(4 * wp.P + 1) * 4) + 15) & ~(size_t)15;
  const size_t frame_bytes = ((size_t)wp.M * (G::K + 1) + kWpf * G::WORK) * sizeof(float2);
  const size_t smem = head + kFpc * frame_bytes + (size_t)wp.S * 16 + 16 * 8 + kWarps * 4 + Phase::smem(mp, wp.S);
  SRPGPU_CHECK_ARG(smem <= 227 * 1024, SRPGPU_ERR_UNSUPPORTED,
                   "%s: %d channels x %d samples per frame and %d TD-GCC samples need %zu B of shared memory",
                   what, wp.M, wp.L, wp.S, smem);
  auto kern = frontend_map_kernel<LP, Phase, kWpf>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("%s: cannot reserve %zu B shared memory", what, smem);
    return SRPGPU_ERR_LAUNCH;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>((wp.F + kFpc - 1) / kFpc, (int64_t)num_sms() * per_sm);
  if (grid <= 0) return SRPGPU_OK;
  kern<<<(unsigned)grid, kWarps * 32, smem, st>>>(wp, Phase{mp});
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

// tiny batches (<= 2 frames per SM): a CTA of 4 warps per frame; else 4 frames per CTA
template <int LP, class Phase, class Map>
static int launch_fused(const WarpParams& wp, const Map& mp, cudaStream_t st, const char* what) {
  static const int forced = [] {                      // tuning override: SRPGPU_FUSED_WPF=1|2|4
    const char* v = std::getenv("SRPGPU_FUSED_WPF");
    return v ? std::atoi(v) : 0;
  }();
  if (forced == 2) return launch_fused_w<LP, Phase, 2>(wp, mp, st, what);
  if (forced == 4 || (forced != 1 && wp.F <= 2 * (int64_t)num_sms()))
    return launch_fused_w<LP, Phase, 4>(wp, mp, st, what);
  return launch_fused_w<LP, Phase, 1>(wp, mp, st, what);
}

template <int LP, int OUT, int kWpf>
static int launch(const WarpParams& wp, cudaStream_t st, const char* what) {
  using G = Geo<LP>;
  const size_t head = (((size_t)32 * LP * 8 + (size_t)(4 * wp.P + 1 + kWarps) * 4) + 15) & ~(size_t)15;
  const size_t frame_bytes = ((size_t)wp.M * (G::K + 1) + kWpf * G::WORK) * sizeof(float2);
  const size_t smem = head + (kWarps / kWpf) * frame_bytes;
  if (smem > 227 * 1024) return 1;   // caller falls back to the block kernel
  auto kern = frontend_warp_kernel<LP, OUT, kWpf>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("%s: cannot reserve %zu B shared memory", what, smem);
    return SRPGPU_ERR_LAUNCH;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  if (per_sm < 1) return 1;
  const int64_t need = (wp.F + kWarps / kWpf - 1) / (kWarps / kWpf);
  const int64_t grid = std::min<int64_t>(need, (int64_t)num_sms() * per_sm);
  if (grid <= 0) return SRPGPU_OK;
  kern<<<(unsigned)grid, kWarps * 32, smem, st>>>(wp);
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

template <int OUT, int kWpf>
static int by_len(const WarpParams& wp, cudaStream_t st, const char* what) {
  switch (wp.L) {
    case 256: return launch<8, OUT, kWpf>(wp, st, what);
    case 512: return launch<16, OUT, kWpf>(wp, st, what);
    case 1024: return launch<32, OUT, kWpf>(wp, st, what);
    default: return 1;
  }
}

}  // namespace wf

// Returns 0 on launch, 1 if the shape is not covered (caller uses the block kernel),
// a negative status on error.
int frontend_sspi_launch(const WarpParams& wp, const SellMap& mp, cudaStream_t st, const char* what) {
  switch (wp.L) {
    case 256: return wf::launch_fused<8, wf::SellPhase>(wp, mp, st, what);
    case 512: return wf::launch_fused<16, wf::SellPhase>(wp, mp, st, what);
    case 1024: return wf::launch_fused<32, wf::SellPhase>(wp, mp, st, what);
    default:
      set_error("%s: the fused chain needs a frame length of 256, 512 or 1024 (got %d)", what, wp.L);
      return SRPGPU_ERR_UNSUPPORTED;
  }
}

int frontend_slri_launch(const WarpParams& wp, const SlriMap& mp, cudaStream_t st, const char* what) {
  switch (wp.L) {
    case 256: return wf::launch_fused<8, wf::SlriPhase>(wp, mp, st, what);
    case 512: return wf::launch_fused<16, wf::SlriPhase>(wp, mp, st, what);
    case 1024: return wf::launch_fused<32, wf::SlriPhase>(wp, mp, st, what);
    default:
      set_error("%s: the fused chain needs a frame length of 256, 512 or 1024 (got %d)", what, wp.L);
      return SRPGPU_ERR_UNSUPPORTED;
  }
}

int frontend_warp_launch(const WarpParams& wp, int out, cudaStream_t st, const char* what) {
  // warps per frame (measured on B200, graph replays): a CTA of 4 warps per frame for
  // tiny batches (cfg1, 100 frames: 25 -> 15 us; the frame's FFT rounds run side by side),
  // a warp per frame while frames still fit in one wave of warps (cfg2: 29 us vs 35 with
  // 2 or 4), two warps per frame for large batches (cfg3 10^4 frames: 344 vs 414 us)
  const int64_t sms = num_sms();
  const int kw = wp.F <= 2 * sms ? 4 : (wp.F <= 8 * sms ? 1 : 2);
  if (out == W_OUT_GCC)
    return kw == 4 ? wf::by_len<W_OUT_GCC, 4>(wp, st, what)
                   : kw == 1 ? wf::by_len<W_OUT_GCC, 1>(wp, st, what) : wf::by_len<W_OUT_GCC, 2>(wp, st, what);
  if (out == W_OUT_XI)
    return kw == 4 ? wf::by_len<W_OUT_XI, 4>(wp, st, what)
                   : kw == 1 ? wf::by_len<W_OUT_XI, 1>(wp, st, what) : wf::by_len<W_OUT_XI, 2>(wp, st, what);
  return 1;
}

}  // namespace srpgpu
