// Task-per-warp frontend for frame lengths L = 64 * Q (Q = 4, 8, 16: L = 256, 512, 1024).
//
// Same math as frontend_warp.cu (stft_frame + fd_gcc, frontend.py:89-160; td_gcc_samples,
// sampling.py:106-134), cut into smaller warp tasks so that a frame's work runs on several
// warps at once.  The warp-per-frame kernel holds 32 complex points per lane (167
// registers) and runs a frame's FFT rounds back to back; at latency-bound batch sizes
// (cfg1/cfg2: 100-1000 frames, i.e. a few warps per SM) the frame latency is the step time.
// Here a CTA owns one frame and its warps take independent tasks:
//   * forward task = one real channel: its L real samples as an N = L/2 point complex FFT
//     (16 points per lane at L = 1024), then the real-spectrum split
//     Y[k] = E[k] + W_L^k O[k] (k = 0..N) into the channel's shared-memory slot;
//   * inverse task = one microphone pair: PHAT cross-spectrum straight into registers,
//     the Hermitian spectrum folded into an N point complex inverse FFT
//     (x[2m] + i x[2m+1] = sum_k (E[k] + i O[k]) W_N^{-km}), and only the kept lags
//     |n| <= N_p evaluated: the first FFT step in registers, the second as a cross-lane
//     transpose-reduction over the few outputs m = floor(n / 2) that are needed.
// The N point FFT is four-step: N = 32 x Q, lane l holds points l + 32 j (j < Q); a Q point
// radix-2 DIF in registers; twiddle W_N^{l a}; the 32 point transforms over l are a
// padded shared-memory transpose, Q point DIFs over every (32/Q)-th lane value and a
// radix-(32/Q) DIF across neighbouring lanes by shuffles.
#include "frontend_warp.cuh"

namespace srpgpu {

namespace lf {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// d * W_32^m for m in [0, 16), m known at compile time after unrolling
__device__ __forceinline__ float2 tw32mul(float2 d, int m) {
  constexpr float c1 = 0.98078528040323043f, s1 = 0.19509032201612825f;
  constexpr float c2 = 0.92387953251128674f, s2 = 0.38268343236508978f;
  constexpr float c3 = 0.83146961230254524f, s3 = 0.55557023301960218f;
  constexpr float c4 = 0.70710678118654752f;
  float2 w;
  switch (m & 15) {
    case 0: return d;
    case 8: return make_float2(d.y, -d.x);
    case 1: w = make_float2(c1, -s1); break;
    case 2: w = make_float2(c2, -s2); break;
    case 3: w = make_float2(c3, -s3); break;
    case 4: w = make_float2(c4, -c4); break;
    case 5: w = make_float2(s3, -c3); break;
    case 6: w = make_float2(s2, -c2); break;
    case 7: w = make_float2(s1, -c1); break;
    case 9: w = make_float2(-s1, -c1); break;
    case 10: w = make_float2(-s2, -c2); break;
    case 11: w = make_float2(-s3, -c3); break;
    case 12: w = make_float2(-c4, -c4); break;
    case 13: w = make_float2(-c3, -s3); break;
    case 14: w = make_float2(-c2, -s2); break;
    default: w = make_float2(-c1, -s1); break;
  }
  return cmul(d, w);
}

// radix-2 DIF over Q points in registers: natural order in, v[i] = X[brev_Q(i)] out
template <int Q>
__device__ __forceinline__ void dif(float2 (&v)[Q]) {
#pragma unroll
  for (int h = Q / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int b = 0; b < Q; b += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 a = v[b + j], c = v[b + j + h];
        v[b + j] = cadd(a, c);
        v[b + j + h] = tw32mul(csub(a, c), j * (16 / h));   // W_{2h}^j
      }
    }
  }
}

template <int Q>
__host__ __device__ constexpr int brev(int i) {
  int r = 0;
  for (int b = 1, o = Q >> 1; b < Q; b <<= 1, o >>= 1)
    if (i & b) r |= o;
  return r;
}

template <int Q>
struct Geo {
  static constexpr int N = 32 * Q;      // complex FFT length (= K = half_len)
  static constexpr int L = 2 * N;       // frame length
  static constexpr int E = 32 / Q;      // lanes per second-step transform
  static constexpr int RS = 32 + E;     // transpose row stride (float2): conflict-free writes and reads
  static constexpr int SLOT = N + 32;   // float2 per channel slot (>= Q * RS, >= N + 1, >= padded Z)
};

// padded position of Z[k] in a slot: the Q*Q blocks of the cross-lane outputs are shifted
// by 16/E float2 so the natural-order writes of one half-warp hit distinct banks
template <int Q>
__device__ __forceinline__ int zpos(int k) {
  return k + (16 / Geo<Q>::E) * (k / (Q * Q));
}

struct Tables {
  const float2* twA;    // [Q][32]  W_N^{l a}
  const float2* twL;    // [N]      W_L^k
  const float2* tw32;   // [32]     W_32^m
};

// Forward task: channel c of the frame starting at `start` -> Y[0..N] in slot; adds sum |Y|^2.
template <int Q>
__device__ __forceinline__ void forward_channel(const WarpParams& prm, int c, int64_t start, float2* slot,
                                                const Tables& t, int lane, float& energy) {
  using G = Geo<Q>;
  constexpr int N = G::N, E = G::E, RS = G::RS;
  const float* x = prm.samples + (int64_t)c * prm.ld_samples + start;
  const float2* w2 = reinterpret_cast<const float2*>(prm.window);
  float2 v[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const int m = lane + 32 * j;                       // z[m] = x[2m] + i x[2m+1]
    const float2 w = __ldg(w2 + m);
    v[j] = make_float2(__ldg(x + 2 * m) * w.x, __ldg(x + 2 * m + 1) * w.y);
  }
  dif<Q>(v);                                           // v[i] = A_l[brev(i)]
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int a = brev<Q>(i);
    slot[a * RS + lane] = cmul(v[i], t.twA[a * 32 + lane]);
  }
  __syncwarp();
  const int a = lane / E, e = lane % E;
#pragma unroll
  for (int q = 0; q < Q; ++q) v[q] = slot[a * RS + e + E * q];
  dif<Q>(v);                                           // v[i] = C_{a,e}[brev(i)]
  if (E > 1) {
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = cmul(v[i], t.tw32[(e * brev<Q>(i)) & 31]);   // W_32^{e b0}
  }
  // radix-E DIF across the E neighbouring lanes of the same a
#pragma unroll
  for (int h = E / 2; h >= 1; h >>= 1) {
    const bool up = (e & h) != 0;
    const float2 w = up ? t.tw32[(e & (h - 1)) * (16 / h)] : make_float2(1.f, 0.f);   // W_{2h}^{e mod h}
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      float2 p;
      p.x = __shfl_xor_sync(0xffffffffu, v[i].x, h);
      p.y = __shfl_xor_sync(0xffffffffu, v[i].y, h);
      v[i] = up ? cmul(csub(p, v[i]), w) : cadd(v[i], p);
    }
  }
  int tq = 0;                                          // this lane's output block: brev_E(e)
#pragma unroll
  for (int b = 1, o = E >> 1; b < E; b <<= 1, o >>= 1)
    if (e & b) tq |= o;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < Q; ++i) slot[zpos<Q>(a + Q * brev<Q>(i) + Q * Q * tq)] = v[i];   // Z[k], natural k
  __syncwarp();
  // real-spectrum split (Y = E + W_L^k O) for k = lane + 32 i, and k = N on lane 0
  float2 y[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int k = lane + 32 * i;
    const float2 zk = slot[zpos<Q>(k)];
    const float2 zn = slot[zpos<Q>((N - k) & (N - 1))];
    const float2 ev = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
    const float2 od = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
    y[i] = cadd(ev, cmul(t.twL[k], od));
    energy += y[i].x * y[i].x + y[i].y * y[i].y;
  }
  float yN = 0.f;
  if (lane == 0) {
    const float2 z0 = slot[zpos<Q>(0)];
    yN = z0.x - z0.y;
    energy += yN * yN;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < Q; ++i) slot[lane + 32 * i] = y[i];
  if (lane == 0) slot[N] = make_float2(yN, 0.f);
}

// Sum of 32 R floats over the warp's lanes: lane l ends with the sums of v[l R .. l R + R).
template <int R>
__device__ __forceinline__ void transpose_reduce(float (&v)[32 * R], int lane) {
#pragma unroll
  for (int o = 16, half = 16 * R; o >= 1; o >>= 1, half >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = up ? v[i + half] : v[i];
      const float send = up ? v[i] : v[i + half];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// Inverse task: pair p's PHAT cross-spectrum -> its kept TD-GCC lags |n| <= Np.
template <int Q>
__device__ __forceinline__ void inverse_pair(const WarpParams& prm, const float2* ya, const float2* yb, const Phat& ph,
                                             const Tables& t, int lane, int Np, int off, int64_t f, float* dst,
                                             int64_t sst) {
  using G = Geo<Q>;
  constexpr int CB = 16 / Q;                           // second-step blocks per reduction
  constexpr int NF = 2 * Q * CB, R = NF / 32;          // 32 floats reduced per chunk, one per lane
  float2 ps[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const int k = lane + 32 * j;
    ps[j] = (k == 0) ? make_float2(0.f, 0.f) : ph(cmulc(ya[k], yb[k]));
  }
  // Psi[N - k]: lane 32 - l, register Q - 1 - j (lane 0: its own register Q - j, Psi[N] = 0)
  const int src = (32 - lane) & 31;
  float2 pn[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    pn[j].x = __shfl_sync(0xffffffffu, ps[Q - 1 - j].x, src);
    pn[j].y = __shfl_sync(0xffffffffu, ps[Q - 1 - j].y, src);
  }
  const bool l0 = lane == 0;
#pragma unroll
  for (int j = Q - 1; j >= 1; --j) pn[j] = l0 ? pn[j - 1] : pn[j];
  if (l0) pn[0] = make_float2(0.f, 0.f);
  // conj of the folded input Z[k] = E[k] + i W_L^{-k} D[k], E = P + conj Pn, D = P - conj Pn
  float2 v[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const int k = lane + 32 * j;
    const float2 ev = make_float2(ps[j].x + pn[j].x, ps[j].y - pn[j].y);
    const float2 dv = make_float2(ps[j].x - pn[j].x, ps[j].y + pn[j].y);
    const float2 od = cmulc(dv, t.twL[k]);
    v[j] = make_float2(ev.x - od.y, -(ev.y + od.x));
  }
  dif<Q>(v);                                           // v[i] = conj(A_l[brev(i)])
#pragma unroll
  for (int a = 0; a < Q; ++a) {                        // in place: v[brev(a)] = conj(A_l[a]) W_N^{l a}
    const int i = brev<Q>(a);
    v[i] = cmul(v[i], t.twA[a * 32 + lane]);
  }
  // outputs m = a + Q c for the kept lags: m = floor(n / 2) in [-ceil(Np/2), floor(Np/2)];
  // conj z[m] = sum_l conj(A_l[a]) W_N^{l a} W_32^{l c}, CB values of c per reduction
  const int cmin = -(((Np + 1) / 2 + Q - 1) / Q), cmax = (Np / 2) / Q;
  for (int c0 = cmin; c0 <= cmax; c0 += CB) {
    float vals[NF];
#pragma unroll
    for (int ci = 0; ci < CB; ++ci) {
      const float2 w = t.tw32[(lane * (c0 + ci)) & 31];   // W_32^{l c}
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        const float2 r = cmul(v[brev<Q>(a)], w);
        vals[(a * CB + ci) * 2] = r.x;
        vals[(a * CB + ci) * 2 + 1] = r.y;
      }
    }
    transpose_reduce<R>(vals, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int fi = lane * R + r;
      const int s = fi >> 1, ri = fi & 1;
      const int m = s / CB + Q * (c0 + s % CB);
      const int n = 2 * m + ri;                        // x[2m] = Re z[m], x[2m+1] = Im z[m]
      if (n >= -Np && n <= Np) {
        const int d = n >= 0 ? n : 2 * Np + 1 + n;     // reference lag order 0..N_p, -N_p..-1
        put_xi(prm, dst, sst, f, off, Np, d, ri ? -vals[r] : vals[r]);
      }
    }
  }
}

// resident CTAs per SM the register budget is cut for: the kernel is issue / latency bound
// with few warps (ncu cfg4: 8 warps per SM, 55% issue active), so a second (third) CTA per
// SM pays more than the registers it costs -- cfg4 (Q = 16, 2 CTAs at 128 registers, no
// spills; 80 KB of shared memory each) 3.36 -> 2.64 ms per 10^4 frames; Q = 8 fits 3 at
// 80 registers without spills
#ifndef LANE_MINB
#define LANE_MINB(Q) ((Q) >= 16 ? 2 : 3)
#endif

template <int Q, int OUT, int WPF>
__global__ void __launch_bounds__(WPF * 32, LANE_MINB(Q))
frontend_lane_kernel(const WarpParams prm) {
  using G = Geo<Q>;
  constexpr int N = G::N, L = G::L, K = N, B = K - 1, SLOT = G::SLOT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* twA = reinterpret_cast<float2*>(smem_raw);   // [Q][32]
  float2* twL = twA + Q * 32;                          // [N]
  float2* tw32 = twL + N;                              // [32]
  int* s_pairs = reinterpret_cast<int*>(tw32 + 32);    // [2P]
  int* s_counts = s_pairs + 2 * prm.P;                 // [P]
  int* s_off = s_counts + prm.P;                       // [P+1]
  float* s_energy = reinterpret_cast<float*>(s_off + prm.P + 1);   // [WPF]
  const size_t head = ((size_t)(Q * 32 + N + 32) * 8 + (size_t)(4 * prm.P + 1 + WPF) * 4 + 15) & ~(size_t)15;
  float2* spec = reinterpret_cast<float2*>(smem_raw + head);       // [M][SLOT]
  const int M = prm.M, P = prm.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  for (int e = threadIdx.x; e < Q * 32; e += blockDim.x) {
    float sn, cs;
    sincospif(2.0f * (float)((e >> 5) * (e & 31)) / (float)N, &sn, &cs);
    twA[e] = make_float2(cs, -sn);
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    float sn, cs;
    sincospif(2.0f * (float)k / (float)L, &sn, &cs);
    twL[k] = make_float2(cs, -sn);
  }
  if (threadIdx.x < 32) {
    float sn, cs;
    sincospif((float)threadIdx.x / 16.0f, &sn, &cs);
    tw32[threadIdx.x] = make_float2(cs, -sn);
  }
  for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) s_pairs[i] = prm.pairs[i];
  if (OUT == W_OUT_XI) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_counts[i] = prm.counts[i];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) s_off[i] = prm.offsets[i];
  }
  __syncthreads();
  const Tables t = {twA, twL, tw32};

  for (int64_t f = blockIdx.x; f < prm.F; f += gridDim.x) {
    const int64_t start = (prm.first_frame + f) * (int64_t)prm.hop;
    float energy = 0.f;
    for (int c = wid; c < M; c += WPF) forward_channel<Q>(prm, c, start, spec + (size_t)c * SLOT, t, lane, energy);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
    if (lane == 0) s_energy[wid] = energy;
    __syncthreads();                                   // spectra + energy of the frame complete
    float floor = prm.floor_value;
    if (prm.weighting && prm.floor_mode == 0) {
      float e = 0.f;
#pragma unroll
      for (int w = 0; w < WPF; ++w) e += s_energy[w];
      floor = prm.floor_value * e;
    }
    const Phat ph(prm.weighting, floor);
    if (OUT == W_OUT_GCC) {
      float2* dst = prm.gcc_out + f * prm.gcc_ld;
      for (int p = wid; p < P; p += WPF) {
        const float2* ya = spec + (size_t)s_pairs[2 * p] * SLOT;
        const float2* yb = spec + (size_t)s_pairs[2 * p + 1] * SLOT;
        for (int k = 1 + lane; k < K; k += 32) {
          float2 val = ph(cmulc(ya[k], yb[k]));
          if (prm.round_tf32) val = make_float2(tf32_rne(val.x), tf32_rne(val.y));
          dst[p * B + k - 1] = val;
        }
      }
      for (int64_t idx = (int64_t)P * B + threadIdx.x; idx < prm.gcc_ld; idx += blockDim.x)
        dst[idx] = make_float2(0.f, 0.f);
    } else {
      float* dst = prm.xi_out + (prm.xi_ld ? f : f * (int64_t)prm.S);
      const int64_t sst = prm.xi_ld ? prm.xi_ld : 1;
      for (int p = wid; p < P; p += WPF)
        inverse_pair<Q>(prm, spec + (size_t)s_pairs[2 * p] * SLOT, spec + (size_t)s_pairs[2 * p + 1] * SLOT,
                           ph, t, lane, s_counts[p], s_off[p], f, dst, sst);
      if (prm.xi_planes && !prm.planes_ld && wid == 0) {   // zero the planes' pad columns [S, cols8)
        uint16_t* pl = prm.xi_planes + f * prm.cols8;
        for (int c = prm.S + lane; c < prm.cols8; c += 32) {
          pl[c] = 0;
          pl[prm.F * prm.cols8 + c] = 0;
        }
      }
    }
    __syncthreads();                                   // spectra free for the next frame
  }
}

template <int Q>
size_t smem_bytes(const WarpParams& wp, int wpf) {
  const size_t head = ((size_t)(Q * 32 + 32 * Q + 32) * 8 + (size_t)(4 * wp.P + 1 + wpf) * 4 + 15) & ~(size_t)15;
  return head + (size_t)wp.M * Geo<Q>::SLOT * sizeof(float2);
}

template <int Q, int OUT, int WPF>
static int launch(const WarpParams& wp, cudaStream_t st, const char* what) {
  const size_t smem = smem_bytes<Q>(wp, WPF);
  if (smem > 227 * 1024) return 1;
  auto kern = frontend_lane_kernel<Q, OUT, WPF>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("%s: cannot reserve %zu B shared memory", what, smem);
    return SRPGPU_ERR_LAUNCH;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPF * 32, smem);
  if (per_sm < 1) return 1;
  const int64_t grid = std::min<int64_t>(wp.F, (int64_t)num_sms() * per_sm);
  if (grid <= 0) return SRPGPU_OK;
  kern<<<(unsigned)grid, WPF * 32, smem, st>>>(wp);
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

// warps per frame: one round of forward tasks for up to 4 channels, else 8 warps
template <int Q, int OUT>
static int by_m(const WarpParams& wp, cudaStream_t st, const char* what) {
  return wp.M <= 4 ? launch<Q, OUT, 4>(wp, st, what) : launch<Q, OUT, 8>(wp, st, what);
}

}  // namespace lf

int frontend_lane_launch(const WarpParams& wp, int out, cudaStream_t st, const char* what) {
  const int Q = wp.L / 64;
  if (wp.L != 64 * Q || (Q != 4 && Q != 8 && Q != 16) || wp.K != wp.L / 2) return 1;
  if (Q == 4) return out == W_OUT_GCC ? lf::by_m<4, W_OUT_GCC>(wp, st, what) : lf::by_m<4, W_OUT_XI>(wp, st, what);
  if (Q == 8) return out == W_OUT_GCC ? lf::by_m<8, W_OUT_GCC>(wp, st, what) : lf::by_m<8, W_OUT_XI>(wp, st, what);
  return out == W_OUT_GCC ? lf::by_m<16, W_OUT_GCC>(wp, st, what) : lf::by_m<16, W_OUT_XI>(wp, st, what);
}

}  // namespace srpgpu
