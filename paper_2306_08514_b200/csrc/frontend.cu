// Frontend of the SRP-map hot path on sm_100a:
//   samples --(windowed real FFT)--> spectra Y[m][0..K]          frontend.py:89-107
//   spectra --(pair products + PHAT)--> psi[p][k], k = 1..K-1     frontend.py:127-160
//   psi --(unnormalized real iFFT, kept lags)--> xi[S]            sampling.py:106-134
//
// One templated kernel family covers every entry (in -> out) combination, so the
// fused chains (samples -> psi, samples -> xi) never write the intermediate
// spectra / cross-spectra to HBM.  A CTA owns one frame at a time (grid-stride
// over frames).  FFTs are radix-2^3 decimation-in-time passes over shared memory
// (8 points per thread in registers per pass: 4 passes at L = 1024, 3 at 512).
// Two real channels are packed into one complex FFT for the forward transform;
// two pairs' Hermitian spectra are packed into one complex FFT for the inverse.
#include "frontend_warp.cuh"

namespace srpgpu {

enum { IN_SAMPLES = 0, IN_SPECTRA = 1, IN_GCC = 2 };
enum { OUT_SPECTRA = 0, OUT_GCC = 1, OUT_XI = 2 };

struct FrontendParams {
  const float* samples;
  int64_t ld_samples;
  const float* window;
  const float2* spectra_in;   // [F][M][K+1]
  const float2* gcc_in;       // [F][P][K-1]
  int32_t M, L, K, log2L, hop;
  int64_t first_frame, F;
  const int32_t* pairs;       // [P][2], device
  int32_t P;
  int32_t weighting;          // 0 none, 1 phat
  int32_t floor_mode;         // 0: floor = floor_value * frame energy; 1: absolute
  float floor_value;
  const int32_t* counts;      // [P], device
  const int32_t* offsets;     // [P+1], device
  int32_t S;
  float2* spectra_out;        // [F][M][K+1]
  float* energy_out;          // [F]
  float2* gcc_out;            // [F][P][K-1]
  float* xi_out;              // [F][S]
  int32_t nbuf;               // concurrent FFT buffers
  int64_t gcc_ld;             // complex elements per frame row of gcc_out (>= P*(K-1))
  int64_t xi_ld;              // 0: xi_out is frame-major [F][S]; > 0: lag-major [S][xi_ld]
  int32_t round_tf32;         // round gcc_out to TF32 (RNE) for the tensor-core map
  uint16_t* xi_planes;        // optional bf16 hi/lo planes [2][F][cols8] (warp path only)
  int32_t cols8;
  int32_t xi_natural;         // planes in natural lag order per pair
  int64_t planes_ld;          // 0: frame-major planes; > 0: lag-major [2][cols8][planes_ld]
  int32_t planes_tf32;        // fp32 hi / lo TF32 planes instead of bf16 (lag-major only)
  int32_t* warp_used;         // set to 1 when the warp-per-frame kernel ran
};

constexpr int kFrontThreads = 256;

// One DIT pass of R radix-2 stages starting at stage s0 over nb buffers of L points.
template <int R>
__device__ __forceinline__ void fft_pass(float2* __restrict__ buf, int nb, int L, int log2L, int s0,
                                         const float2* __restrict__ tw) {
  constexpr int G = 1 << R;
  const int h0 = 1 << s0;
  const int log2_groups = log2L - R;
  const int total = nb << log2_groups;
  for (int g = threadIdx.x; g < total; g += blockDim.x) {
    const int b = g >> log2_groups;
    const int gi = g & ((1 << log2_groups) - 1);
    const int t = gi & (h0 - 1);
    const int blk = gi >> s0;
    float2* base = buf + (size_t)b * L + (blk << (s0 + R)) + t;
    float2 e[G];
#pragma unroll
    for (int m = 0; m < G; ++m) e[m] = base[m * h0];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int tw_shift = log2L - s0 - q - 1;
#pragma unroll
      for (int m = 0; m < G; ++m) {
        if (m & (1 << q)) continue;
        const int j = t + (m & ((1 << q) - 1)) * h0;
        const float2 w = tw[j << tw_shift];
        const float2 u = e[m];
        const float2 v = cmul(e[m | (1 << q)], w);
        e[m] = make_float2(u.x + v.x, u.y + v.y);
        e[m | (1 << q)] = make_float2(u.x - v.x, u.y - v.y);
      }
    }
#pragma unroll
    for (int m = 0; m < G; ++m) base[m * h0] = e[m];
  }
}

// Forward DFT (sign -1) of nb buffers whose inputs were stored bit-reversed.
__device__ void block_fft(float2* buf, int nb, int L, int log2L, const float2* tw) {
  int s = 0;
  while (log2L - s >= 3) {
    fft_pass<3>(buf, nb, L, log2L, s, tw);
    s += 3;
    __syncthreads();
  }
  if (log2L - s == 2) {
    fft_pass<2>(buf, nb, L, log2L, s, tw);
    __syncthreads();
  } else if (log2L - s == 1) {
    fft_pass<1>(buf, nb, L, log2L, s, tw);
    __syncthreads();
  }
}

__device__ __forceinline__ int bitrev(int n, int log2L) {
  return (int)(__brev((unsigned)n) >> (32 - log2L));
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float total = 0.f;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) total += red[w];
  return total;
}

// PHAT-weighted cross-spectrum of pair (m, m') at bin k (frontend.py:152-158).
__device__ __forceinline__ float2 cross_bin(const float2* spec, int Kp1, int m, int mp, int k,
                                            int weighting, float floor) {
  const float2 a = spec[m * Kp1 + k];
  const float2 b = spec[mp * Kp1 + k];
  float2 raw = cmulc(a, b);
  if (weighting) {
    // raw / max(|raw|, floor), 0 where that is 0 (frontend.py:154-158)
    const float mag2 = raw.x * raw.x + raw.y * raw.y;
    const float inv = (mag2 > floor * floor && mag2 > 0.f) ? rsqrtf(mag2) : (floor > 0.f ? 1.0f / floor : 0.f);
    raw.x *= inv;
    raw.y *= inv;
  }
  return raw;
}

template <int IN, int OUT>
__global__ void __launch_bounds__(kFrontThreads)
frontend_kernel(const FrontendParams prm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = prm.L, K = prm.K, log2L = prm.log2L, M = prm.M, P = prm.P;
  const int Kp1 = K + 1, B = K - 1;
  float2* tw = reinterpret_cast<float2*>(smem_raw);                 // [L/2]
  float2* fft = tw + (L >> 1);                                         // [nbuf][L]
  float2* spec = fft + (size_t)prm.nbuf * L;                           // [M][K+1]
  const bool need_spec = (IN != IN_GCC);
  int* s_pairs = reinterpret_cast<int*>(spec + (need_spec ? (size_t)M * Kp1 : 0));  // [2P]
  int* s_counts = s_pairs + 2 * P;                                     // [P]
  int* s_off = s_counts + P;                                           // [P+1]
  float* red = reinterpret_cast<float*>(s_off + P + 1);                // [32]

  for (int n = threadIdx.x; n < (L >> 1); n += blockDim.x) {
    float s, c;
    sincospif(2.0f * (float)n / (float)L, &s, &c);
    tw[n] = make_float2(c, -s);
  }
  if (OUT != OUT_SPECTRA || IN == IN_GCC) {
    for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) s_pairs[i] = prm.pairs ? prm.pairs[i] : 0;
  }
  if (OUT == OUT_XI) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_counts[i] = prm.counts[i];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) s_off[i] = prm.offsets[i];
  }
  __syncthreads();

  for (int64_t f = blockIdx.x; f < prm.F; f += gridDim.x) {
    float energy = 0.f;
    // ---------------- phase A: spectra of all channels ----------------
    if (IN == IN_SAMPLES) {
      const int64_t start = (prm.first_frame + f) * (int64_t)prm.hop;
      for (int ch0 = 0; ch0 < M; ch0 += 2 * prm.nbuf) {
        const int nb = min(prm.nbuf, (M - ch0 + 1) >> 1);
        for (int idx = threadIdx.x; idx < nb * L; idx += blockDim.x) {
          const int b = idx >> log2L, n = idx & (L - 1);
          const int a = ch0 + 2 * b, c = a + 1;
          const float w = __ldg(prm.window + n);
          const float xa = __ldg(prm.samples + (int64_t)a * prm.ld_samples + start + n) * w;
          const float xb = (c < M) ? __ldg(prm.samples + (int64_t)c * prm.ld_samples + start + n) * w : 0.f;
          fft[(size_t)b * L + bitrev(n, log2L)] = make_float2(xa, xb);
        }
        __syncthreads();
        block_fft(fft, nb, L, log2L, tw);
        for (int idx = threadIdx.x; idx < nb * Kp1; idx += blockDim.x) {
          const int b = idx / Kp1, k = idx - b * Kp1;
          const int a = ch0 + 2 * b, c = a + 1;
          const float2 Z = fft[(size_t)b * L + k];
          const float2 Zc = conjf2(fft[(size_t)b * L + ((L - k) & (L - 1))]);
          const float2 Xa = make_float2(0.5f * (Z.x + Zc.x), 0.5f * (Z.y + Zc.y));
          spec[a * Kp1 + k] = Xa;
          energy += Xa.x * Xa.x + Xa.y * Xa.y;
          if (c < M) {
            const float2 Xb = make_float2(0.5f * (Z.y - Zc.y), -0.5f * (Z.x - Zc.x));
            spec[c * Kp1 + k] = Xb;
            energy += Xb.x * Xb.x + Xb.y * Xb.y;
          }
        }
        __syncthreads();
      }
    } else if (IN == IN_SPECTRA) {
      const float2* src = prm.spectra_in + f * (int64_t)M * Kp1;
      for (int idx = threadIdx.x; idx < M * Kp1; idx += blockDim.x) {
        const float2 v = src[idx];
        spec[idx] = v;
        energy += v.x * v.x + v.y * v.y;
      }
      __syncthreads();
    }

    float floor = prm.floor_value;
    const bool need_energy = (OUT == OUT_SPECTRA && prm.energy_out) ||
                             (IN != IN_GCC && OUT != OUT_SPECTRA && prm.weighting && prm.floor_mode == 0);
    if (need_energy) {
      energy = block_sum(energy, red);
      if (prm.floor_mode == 0) floor = prm.floor_value * energy;
    }

    // ---------------- phase B: outputs ----------------
    if (OUT == OUT_SPECTRA) {
      float2* dst = prm.spectra_out + f * (int64_t)M * Kp1;
      for (int idx = threadIdx.x; idx < M * Kp1; idx += blockDim.x) dst[idx] = spec[idx];
      if (prm.energy_out && threadIdx.x == 0) prm.energy_out[f] = energy;
    } else if (OUT == OUT_GCC) {
      float2* dst = prm.gcc_out + f * prm.gcc_ld;
      for (int idx = threadIdx.x; idx < P * B; idx += blockDim.x) {
        const int p = idx / B, k = idx - p * B + 1;
        float2 v = cross_bin(spec, Kp1, s_pairs[2 * p], s_pairs[2 * p + 1], k, prm.weighting, floor);
        if (prm.round_tf32) v = make_float2(tf32_rne(v.x), tf32_rne(v.y));
        dst[idx] = v;
      }
      for (int64_t idx = P * B + threadIdx.x; idx < prm.gcc_ld; idx += blockDim.x)
        dst[idx] = make_float2(0.f, 0.f);   // pitch padding
    } else {  // OUT_XI
      const float2* gsrc = (IN == IN_GCC) ? prm.gcc_in + f * (int64_t)P * B : nullptr;
      float* dst = prm.xi_out + (prm.xi_ld ? f : f * (int64_t)prm.S);
      const int64_t sst = prm.xi_ld ? prm.xi_ld : 1;
      for (int p0 = 0; p0 < P; p0 += 2 * prm.nbuf) {
        const int nb = min(prm.nbuf, (P - p0 + 1) >> 1);
        // two-sided spectra Z = Psi_a + j Psi_b (Hermitian extension, bins 0 and K zero),
        // stored conjugated and bit-reversed: x = conj(FFT(conj(Z))) is the unnormalized iDFT.
        for (int idx = threadIdx.x; idx < nb * K; idx += blockDim.x) {
          const int b = idx / K, k = idx - b * K;
          const int pa = p0 + 2 * b, pb = pa + 1;
          float2* fb = fft + (size_t)b * L;
          if (k == 0) {
            fb[bitrev(0, log2L)] = make_float2(0.f, 0.f);
            fb[bitrev(K, log2L)] = make_float2(0.f, 0.f);
            continue;
          }
          float2 a, c;
          if (IN == IN_GCC) {
            a = gsrc[(int64_t)pa * B + k - 1];
            c = (pb < P) ? gsrc[(int64_t)pb * B + k - 1] : make_float2(0.f, 0.f);
          } else {
            a = cross_bin(spec, Kp1, s_pairs[2 * pa], s_pairs[2 * pa + 1], k, prm.weighting, floor);
            c = (pb < P) ? cross_bin(spec, Kp1, s_pairs[2 * pb], s_pairs[2 * pb + 1], k, prm.weighting, floor)
                         : make_float2(0.f, 0.f);
          }
          // Z[k] = a + j c ; Z[L-k] = conj(a) + j conj(c)
          const float2 zk = make_float2(a.x - c.y, a.y + c.x);
          const float2 zn = make_float2(a.x + c.y, -a.y + c.x);
          fb[bitrev(k, log2L)] = conjf2(zk);
          fb[bitrev(L - k, log2L)] = conjf2(zn);
        }
        __syncthreads();
        block_fft(fft, nb, L, log2L, tw);
        // keep lags 0..N_p, then -N_p..-1 (sampling.py:62-65,126-133)
        const int s_lo = s_off[p0];
        const int s_hi = s_off[min(P, p0 + 2 * nb)];
        for (int s = s_lo + threadIdx.x; s < s_hi; s += blockDim.x) {
          int q = p0;
          while (s_off[q + 1] <= s) ++q;
          const int c = s_counts[q];
          const int j = s - s_off[q];
          const int n = (j <= c) ? j : L - (2 * c + 1 - j);
          const float2 v = fft[(size_t)((q - p0) >> 1) * L + n];
          dst[s * sst] = ((q - p0) & 1) ? -v.y : v.x;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

static size_t frontend_smem(int in, int out, int L, int K, int M, int P, int nbuf) {
  size_t b = (size_t)(L / 2) * sizeof(float2) + (size_t)nbuf * L * sizeof(float2);
  if (in != IN_GCC) b += (size_t)M * (K + 1) * sizeof(float2);
  b += (size_t)(2 * P + P + P + 1) * sizeof(int) + 32 * sizeof(float);
  return (b + 15) & ~(size_t)15;
}

// The task-per-warp kernel (frontend_lane.cu) wins on tiny batches (cfg1, 100 frames: 15 vs
// 17 us; cfg3 geometry, 1000 frames: 53 vs 61 us) and on many channels / long lag windows
// (cfg4, M = 16, N_p up to 58: 2.6 vs 10.4 ms per 10^4 frames); the warp-per-frame kernel
// wins at cfg2 (1000 frames: 33 vs 39 us) and on large batches (cfg3, 10^4 frames: 0.38 vs
// 0.43 ms), medians of 5 alternating runs (tools/bench_frontend.py --rounds 5).
constexpr int64_t kLaneMaxFrames = 2;    // frames per SM (M < 8)
constexpr int64_t kLaneMaxFrames8 = 12;  // frames per SM (M >= 8)
constexpr int kLaneMinMics = 8;     // (r2: with TF32 planes the task kernel wins at every cfg3 batch size)

template <int IN, int OUT>
static int launch_frontend(FrontendParams prm, cudaStream_t stream, const char* what) {
  if (IN == IN_SAMPLES && OUT != OUT_SPECTRA && prm.F > 0) {
    // warp-per-frame register FFT path (frame lengths 256 / 512 / 1024)
    WarpParams wp = {};
    wp.samples = prm.samples; wp.ld_samples = prm.ld_samples; wp.window = prm.window;
    wp.M = prm.M; wp.L = prm.L; wp.K = prm.K; wp.hop = prm.hop;
    wp.first_frame = prm.first_frame; wp.F = prm.F; wp.pairs = prm.pairs; wp.P = prm.P;
    wp.weighting = prm.weighting; wp.floor_mode = prm.floor_mode; wp.floor_value = prm.floor_value;
    wp.counts = prm.counts; wp.offsets = prm.offsets; wp.S = prm.S;
    wp.gcc_out = prm.gcc_out; wp.gcc_ld = prm.gcc_ld; wp.round_tf32 = prm.round_tf32;
    wp.xi_out = prm.xi_out; wp.xi_ld = prm.xi_ld;
    wp.xi_planes = prm.xi_planes; wp.cols8 = prm.cols8; wp.xi_natural = prm.xi_natural;
    wp.planes_ld = prm.planes_ld; wp.planes_tf32 = prm.planes_tf32;
    const int wout = OUT == OUT_GCC ? W_OUT_GCC : W_OUT_XI;
    const int choice = frontend_kernel_choice();
    int r = 1;
    const int64_t lane_frames = (prm.M >= 8 ? kLaneMaxFrames8 : kLaneMaxFrames) * (int64_t)num_sms();
    if (choice == 2 || (choice == 0 && (prm.F <= lane_frames || prm.M >= kLaneMinMics)))
      r = frontend_lane_launch(wp, wout, stream, what);
    if (r == 1 && choice != 3) r = frontend_warp_launch(wp, wout, stream, what);
    if (r == 0 && prm.warp_used) *prm.warp_used = 1;
    if (r <= 0) return r;
  }
  const int need = (OUT == OUT_XI) ? (prm.P + 1) / 2 : (IN == IN_SAMPLES ? (prm.M + 1) / 2 : 0);
  const size_t budget = 200 * 1024;
  int nbuf = max(1, need);
  while (nbuf > 1 && frontend_smem(IN, OUT, prm.L, prm.K, prm.M, prm.P, nbuf) > budget) --nbuf;
  // prefer leaving room for >= 2 CTAs per SM when the buffers can be split into rounds
  while (nbuf > 2 && frontend_smem(IN, OUT, prm.L, prm.K, prm.M, prm.P, nbuf) > 100 * 1024) --nbuf;
  prm.nbuf = nbuf;
  const size_t smem = frontend_smem(IN, OUT, prm.L, prm.K, prm.M, prm.P, nbuf);
  SRPGPU_CHECK_ARG(smem <= 227 * 1024, SRPGPU_ERR_UNSUPPORTED,
                   "%s: frame of %d samples x %d channels needs %zu B of shared memory", what,
                   prm.L, prm.M, smem);
  auto kern = frontend_kernel<IN, OUT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("%s: cannot reserve %zu B shared memory", what, smem);
    return SRPGPU_ERR_LAUNCH;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFrontThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>(prm.F, (int64_t)num_sms() * per_sm);
  if (grid <= 0) return SRPGPU_OK;
  kern<<<(unsigned)grid, kFrontThreads, smem, stream>>>(prm);
  SRPGPU_CHECK_LAUNCH(what);
  return SRPGPU_OK;
}

static int check_len(int frame_len, int* log2L) {
  if (frame_len < 4 || (frame_len & (frame_len - 1)) != 0 || frame_len > 16384) return 0;
  int l = 0;
  while ((1 << l) < frame_len) ++l;
  *log2L = l;
  return 1;
}

}  // namespace srpgpu

using namespace srpgpu;

static int fill_common(FrontendParams& prm, int32_t frame_len, const char* what,
                       bool need_fft = true) {
  int log2L = 0;
  if (!need_fft && frame_len >= 4 && frame_len % 2 == 0 && frame_len <= 65536) {
    prm.L = frame_len;
    prm.K = frame_len / 2;
    prm.log2L = 0;
    return SRPGPU_OK;
  }
  if (!check_len(frame_len, &log2L)) {
    set_error("%s: frame_len %d is not a power of two in [4, 16384]", what, frame_len);
    return SRPGPU_ERR_UNSUPPORTED;
  }
  prm.L = frame_len;
  prm.K = frame_len / 2;
  prm.log2L = log2L;
  return SRPGPU_OK;
}

static int check_frames(const FrontendParams& prm, int64_t num_samples, const char* what) {
  SRPGPU_CHECK_ARG(prm.hop >= 1, SRPGPU_ERR_VALUE, "%s: hop must be >= 1", what);
  SRPGPU_CHECK_ARG(prm.first_frame >= 0, SRPGPU_ERR_DIMENSION, "%s: negative frame index", what);
  if (prm.F > 0) {
    const int64_t last_end = (prm.first_frame + prm.F - 1) * (int64_t)prm.hop + prm.L;
    SRPGPU_CHECK_ARG(last_end <= num_samples, SRPGPU_ERR_DIMENSION,
                     "%s: frame %lld out of range for %lld samples", what,
                     (long long)(prm.first_frame + prm.F - 1), (long long)num_samples);
  }
  return SRPGPU_OK;
}

extern "C" int srpgpu_stft(const float* samples, int32_t num_channels, int64_t num_samples,
                           int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                           int64_t first_frame, int64_t num_frames, float* spectra, float* energy,
                           srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "stft");
  if (st) return st;
  SRPGPU_CHECK_ARG(num_channels >= 1, SRPGPU_ERR_DIMENSION, "stft: need >= 1 channel");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  prm.spectra_out = reinterpret_cast<float2*>(spectra); prm.energy_out = energy;
  if ((st = check_frames(prm, num_samples, "stft"))) return st;
  return launch_frontend<IN_SAMPLES, OUT_SPECTRA>(prm, as_stream(stream), "stft");
}

extern "C" int srpgpu_fd_gcc(const float* spectra, int64_t num_frames, int32_t num_channels,
                             int32_t half_len, const int32_t* pairs, int32_t num_pairs,
                             int32_t weighting, int32_t floor_mode, double floor_value, float* gcc,
                             srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, 2 * half_len, "fd_gcc", /*need_fft=*/false);
  if (st) return st;
  SRPGPU_CHECK_ARG(half_len >= 2, SRPGPU_ERR_DIMENSION, "fd_gcc: spectra must cover bins 0..2");
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "fd_gcc: unknown weighting");
  prm.spectra_in = reinterpret_cast<const float2*>(spectra);
  prm.F = num_frames; prm.M = num_channels; prm.pairs = pairs; prm.P = num_pairs;
  prm.weighting = weighting; prm.floor_mode = floor_mode; prm.floor_value = (float)floor_value;
  prm.gcc_out = reinterpret_cast<float2*>(gcc);
  prm.gcc_ld = (int64_t)num_pairs * (half_len - 1);
  return launch_frontend<IN_SPECTRA, OUT_GCC>(prm, as_stream(stream), "fd_gcc");
}

extern "C" int srpgpu_gcc_frames(const float* samples, int32_t num_channels, int64_t num_samples,
                                 int64_t ld_samples, const float* window, int32_t frame_len,
                                 int32_t hop, int64_t first_frame, int64_t num_frames,
                                 const int32_t* pairs, int32_t num_pairs, int32_t weighting,
                                 int32_t floor_mode, double floor_value, float* gcc,
                                 int64_t gcc_ld, int32_t flags, srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "gcc_frames");
  if (st) return st;
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "gcc_frames: unknown weighting");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  prm.pairs = pairs; prm.P = num_pairs; prm.weighting = weighting; prm.floor_mode = floor_mode;
  prm.floor_value = (float)floor_value; prm.gcc_out = reinterpret_cast<float2*>(gcc);
  prm.gcc_ld = gcc_ld > 0 ? gcc_ld : (int64_t)num_pairs * (prm.K - 1);
  SRPGPU_CHECK_ARG(prm.gcc_ld >= (int64_t)num_pairs * (prm.K - 1), SRPGPU_ERR_DIMENSION,
                   "gcc_frames: row pitch smaller than P*(K-1)");
  prm.round_tf32 = flags & 1;
  if ((st = check_frames(prm, num_samples, "gcc_frames"))) return st;
  return launch_frontend<IN_SAMPLES, OUT_GCC>(prm, as_stream(stream), "gcc_frames");
}

extern "C" int srpgpu_td_gcc_samples(const float* gcc, int64_t num_frames, int32_t num_pairs,
                                     int32_t half_len, const int32_t* counts, const int32_t* offsets,
                                     int32_t total_samples, float* samples_out, int64_t samples_ld,
                                     srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, 2 * half_len, "td_gcc_samples");
  if (st) return st;
  SRPGPU_CHECK_ARG(half_len >= 2, SRPGPU_ERR_DIMENSION, "td_gcc_samples: half_len must be >= 2");
  prm.gcc_in = reinterpret_cast<const float2*>(gcc);
  prm.F = num_frames; prm.P = num_pairs; prm.counts = counts; prm.offsets = offsets;
  prm.S = total_samples; prm.xi_out = samples_out; prm.xi_ld = samples_ld;
  SRPGPU_CHECK_ARG(samples_ld == 0 || samples_ld >= num_frames, SRPGPU_ERR_DIMENSION,
                   "td_gcc_samples: lag-major pitch smaller than the frame count");
  return launch_frontend<IN_GCC, OUT_XI>(prm, as_stream(stream), "td_gcc_samples");
}

extern "C" int srpgpu_frames_to_samples(const float* samples, int32_t num_channels,
                                        int64_t num_samples, int64_t ld_samples, const float* window,
                                        int32_t frame_len, int32_t hop, int64_t first_frame,
                                        int64_t num_frames, const int32_t* pairs, int32_t num_pairs,
                                        int32_t weighting, int32_t floor_mode, double floor_value,
                                        const int32_t* counts, const int32_t* offsets,
                                        int32_t total_samples, float* samples_out,
                                        int64_t samples_ld, srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "frames_to_samples");
  if (st) return st;
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "frames_to_samples: unknown weighting");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  prm.pairs = pairs; prm.P = num_pairs; prm.weighting = weighting; prm.floor_mode = floor_mode;
  prm.floor_value = (float)floor_value; prm.counts = counts; prm.offsets = offsets;
  prm.S = total_samples; prm.xi_out = samples_out; prm.xi_ld = samples_ld;
  SRPGPU_CHECK_ARG(samples_ld == 0 || samples_ld >= num_frames, SRPGPU_ERR_DIMENSION,
                   "frames_to_samples: lag-major pitch smaller than the frame count");
  if ((st = check_frames(prm, num_samples, "frames_to_samples"))) return st;
  return launch_frontend<IN_SAMPLES, OUT_XI>(prm, as_stream(stream), "frames_to_samples");
}

extern "C" int srpgpu_frames_to_sspi_map(const float* samples, int32_t num_channels, int64_t num_samples,
                                         int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                                         int64_t first_frame, int64_t num_frames, const int32_t* pairs,
                                         int32_t num_pairs, int32_t weighting, int32_t floor_mode,
                                         double floor_value, const int32_t* counts, const int32_t* offsets,
                                         int32_t total_samples, const uint16_t* sell_cols, const float* sell_vals,
                                         const int32_t* sell_chunk_off, int64_t num_candidates, float* z,
                                         int64_t* index, uint64_t* keys, srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "frames_to_sspi_map");
  if (st) return st;
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "frames_to_sspi_map: unknown weighting");
  SRPGPU_CHECK_ARG(num_channels >= 2 && num_pairs >= 1 && total_samples >= 1 && total_samples <= 65535 &&
                       num_candidates >= 1 && num_candidates < (1ll << 31),
                   SRPGPU_ERR_DIMENSION, "frames_to_sspi_map: bad shape");
  SRPGPU_CHECK_ARG(sell_cols && sell_vals && sell_chunk_off, SRPGPU_ERR_VALUE,
                   "frames_to_sspi_map: missing operator arrays");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  if ((st = check_frames(prm, num_samples, "frames_to_sspi_map"))) return st;
  WarpParams wp = {};
  wp.samples = samples; wp.ld_samples = ld_samples; wp.window = window;
  wp.M = num_channels; wp.L = prm.L; wp.K = prm.K; wp.hop = hop;
  wp.first_frame = first_frame; wp.F = num_frames; wp.pairs = pairs; wp.P = num_pairs;
  wp.weighting = weighting; wp.floor_mode = floor_mode; wp.floor_value = (float)floor_value;
  wp.counts = counts; wp.offsets = offsets; wp.S = total_samples;
  SellMap mp = {sell_cols, sell_vals, sell_chunk_off, num_candidates, z, index, keys};
  if (num_frames == 0) return SRPGPU_OK;
  return frontend_sspi_launch(wp, mp, as_stream(stream), "frames_to_sspi_map");
}

extern "C" int srpgpu_frames_to_slri_map(const float* samples, int32_t num_channels, int64_t num_samples,
                                         int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                                         int64_t first_frame, int64_t num_frames, const int32_t* pairs,
                                         int32_t num_pairs, int32_t weighting, int32_t floor_mode,
                                         double floor_value, const int32_t* counts, const int32_t* offsets,
                                         int32_t total_samples, const float* fat, const float* tall_t, int32_t rank,
                                         int64_t num_candidates, float* z, int64_t* index, uint64_t* keys,
                                         srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "frames_to_slri_map");
  if (st) return st;
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "frames_to_slri_map: unknown weighting");
  SRPGPU_CHECK_ARG(num_channels >= 2 && num_pairs >= 1 && total_samples >= 1 && rank >= 1 && rank <= 4096 &&
                       num_candidates >= 1 && num_candidates < (1ll << 31),
                   SRPGPU_ERR_DIMENSION, "frames_to_slri_map: bad shape");
  SRPGPU_CHECK_ARG(fat && tall_t, SRPGPU_ERR_VALUE, "frames_to_slri_map: missing factors");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  if ((st = check_frames(prm, num_samples, "frames_to_slri_map"))) return st;
  WarpParams wp = {};
  wp.samples = samples; wp.ld_samples = ld_samples; wp.window = window;
  wp.M = num_channels; wp.L = prm.L; wp.K = prm.K; wp.hop = hop;
  wp.first_frame = first_frame; wp.F = num_frames; wp.pairs = pairs; wp.P = num_pairs;
  wp.weighting = weighting; wp.floor_mode = floor_mode; wp.floor_value = (float)floor_value;
  wp.counts = counts; wp.offsets = offsets; wp.S = total_samples;
  SlriMap mp = {fat, tall_t, rank, total_samples, num_candidates, z, index, keys};
  if (num_frames == 0) return SRPGPU_OK;
  return frontend_slri_launch(wp, mp, as_stream(stream), "frames_to_slri_map");
}

extern "C" int srpgpu_frames_to_samples_planes(const float* samples, int32_t num_channels,
                                               int64_t num_samples, int64_t ld_samples, const float* window,
                                               int32_t frame_len, int32_t hop, int64_t first_frame,
                                               int64_t num_frames, const int32_t* pairs, int32_t num_pairs,
                                               int32_t weighting, int32_t floor_mode, double floor_value,
                                               const int32_t* counts, const int32_t* offsets,
                                               int32_t total_samples, float* samples_out, int64_t samples_ld,
                                               void* planes, int32_t cols8, int64_t planes_ld, int32_t natural,
                                               const int32_t* natural_src, srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, frame_len, "frames_to_samples");
  if (st) return st;
  SRPGPU_CHECK_ARG(weighting == 0 || weighting == 1, SRPGPU_ERR_VALUE, "frames_to_samples: unknown weighting");
  SRPGPU_CHECK_ARG(planes != nullptr && cols8 >= total_samples && cols8 % 8 == 0 && ((uintptr_t)planes & 15) == 0,
                   SRPGPU_ERR_VALUE, "frames_to_samples: bf16 planes need cols8 >= S, a multiple of 8, 16-byte aligned");
  prm.samples = samples; prm.ld_samples = ld_samples; prm.window = window;
  prm.M = num_channels; prm.hop = hop; prm.first_frame = first_frame; prm.F = num_frames;
  prm.pairs = pairs; prm.P = num_pairs; prm.weighting = weighting; prm.floor_mode = floor_mode;
  prm.floor_value = (float)floor_value; prm.counts = counts; prm.offsets = offsets;
  prm.S = total_samples; prm.xi_out = samples_out; prm.xi_ld = samples_ld;
  prm.xi_planes = reinterpret_cast<uint16_t*>(planes); prm.cols8 = cols8; prm.xi_natural = (natural & 1) ? 1 : 0;
  prm.planes_ld = planes_ld; prm.planes_tf32 = (natural & 4) ? 2 : (natural & 2) ? 1 : 0;
  SRPGPU_CHECK_ARG(!prm.planes_tf32 || planes_ld > 0, SRPGPU_ERR_VALUE,
                   "frames_to_samples: TF32 / fp16 planes are lag-major only (planes_ld > 0)");
  SRPGPU_CHECK_ARG(planes_ld == 0 || (planes_ld >= num_frames && planes_ld % 8 == 0), SRPGPU_ERR_VALUE,
                   "frames_to_samples: lag-major planes need a pitch >= F, a multiple of 8");
  SRPGPU_CHECK_ARG(!natural || natural_src, SRPGPU_ERR_VALUE, "frames_to_samples: natural planes need the column map");
  int32_t warp_used = 0;
  prm.warp_used = &warp_used;
  SRPGPU_CHECK_ARG(samples_ld == 0 || samples_ld >= num_frames, SRPGPU_ERR_DIMENSION,
                   "frames_to_samples: lag-major pitch smaller than the frame count");
  if ((st = check_frames(prm, num_samples, "frames_to_samples"))) return st;
  if ((st = launch_frontend<IN_SAMPLES, OUT_XI>(prm, as_stream(stream), "frames_to_samples"))) return st;
  if (warp_used || num_frames == 0) return SRPGPU_OK;
  // block-kernel frame lengths: split the f32 samples afterwards
  if (prm.planes_tf32 == 2)
    return srpgpu_split_f16_rows(samples_out, samples_ld, total_samples, num_frames,
                                 prm.xi_natural ? natural_src : nullptr, 1.0f, planes, planes_ld, cols8, stream);
  if (prm.planes_tf32)
    return srpgpu_split_tf32_rows(samples_out, samples_ld, total_samples, num_frames,
                                  prm.xi_natural ? natural_src : nullptr, reinterpret_cast<float*>(planes), planes_ld,
                                  cols8, stream);
  if (planes_ld)   // lag-major planes from the lag-major f32 samples
    return srpgpu_split_bf16_rows(samples_out, samples_ld, total_samples, num_frames,
                                  prm.xi_natural ? natural_src : nullptr, planes, planes_ld, cols8, stream);
  return srpgpu_split_bf16_cols(samples_out, samples_ld ? samples_ld : total_samples, samples_ld ? 1 : 0,
                                num_frames, total_samples, prm.xi_natural ? natural_src : nullptr, planes, cols8,
                                stream);
}

extern "C" int srpgpu_spectra_to_samples(const float* spectra, int64_t num_frames,
                                         int32_t num_channels, int32_t half_len,
                                         const int32_t* pairs, int32_t num_pairs, int32_t weighting,
                                         int32_t floor_mode, double floor_value,
                                         const int32_t* counts, const int32_t* offsets,
                                         int32_t total_samples, float* samples_out,
                                         int64_t samples_ld, srpgpu_stream_t stream) {
  FrontendParams prm = {};
  int st = fill_common(prm, 2 * half_len, "spectra_to_samples");
  if (st) return st;
  prm.spectra_in = reinterpret_cast<const float2*>(spectra);
  prm.F = num_frames; prm.M = num_channels; prm.pairs = pairs; prm.P = num_pairs;
  prm.weighting = weighting; prm.floor_mode = floor_mode; prm.floor_value = (float)floor_value;
  prm.counts = counts; prm.offsets = offsets; prm.S = total_samples; prm.xi_out = samples_out;
  prm.xi_ld = samples_ld;
  SRPGPU_CHECK_ARG(samples_ld == 0 || samples_ld >= num_frames, SRPGPU_ERR_DIMENSION,
                   "spectra_to_samples: lag-major pitch smaller than the frame count");
  return launch_frontend<IN_SPECTRA, OUT_XI>(prm, as_stream(stream), "spectra_to_samples");
}
