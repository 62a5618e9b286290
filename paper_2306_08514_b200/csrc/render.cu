// Scene rendering for the sweep command (simulate.py:232-265): every microphone signal is
// the sum over image sources of a 64-tap fractional-delay FIR of the dry source signal,
//   out[m][n] += g_{m,i} sum_t h_{m,i}[t] dry[n - start_{m,i} - t],
// accumulated in image order into a direct-path and a reverberant buffer (float64, as the
// reference renders).  One thread per output sample; the taps, gains and offsets of each
// (microphone, image) are computed on the host exactly as the reference computes them.
#include "common.cuh"

namespace srpgpu {
namespace rnd {

constexpr int kTaps = 64;

__global__ void render_images_kernel(const double* __restrict__ dry, int64_t N, int32_t M, int32_t I,
                                     const int64_t* __restrict__ start, const double* __restrict__ gain,
                                     const double* __restrict__ taps, const int32_t* __restrict__ is_direct,
                                     double* __restrict__ direct, double* __restrict__ reverb) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(idx / N);
    const int64_t n = idx - (int64_t)m * N;
    double d = 0.0, r = 0.0;
    for (int i = 0; i < I; ++i) {
      const int64_t q = n - __ldg(start + (int64_t)m * I + i);     // index into the full convolution
      if (q < 0 || q >= N + kTaps - 1) continue;
      const double* h = taps + ((int64_t)m * I + i) * kTaps;
      double acc = 0.0;
#pragma unroll 8
      for (int t = 0; t < kTaps; ++t) {
        const int64_t j = q - t;
        if (j >= 0 && j < N) acc = fma(__ldg(h + t), __ldg(dry + j), acc);
      }
      acc *= __ldg(gain + (int64_t)m * I + i);
      if (__ldg(is_direct + i)) d += acc;
      else r += acc;
    }
    direct[idx] = d;
    reverb[idx] = r;
  }
}

}  // namespace rnd
}  // namespace srpgpu

using namespace srpgpu;

extern "C" int srpgpu_render_images(const double* dry, int64_t num_samples, int32_t num_mics, int32_t num_images,
                                    const int64_t* start, const double* gain, const double* taps,
                                    const int32_t* is_direct, double* direct, double* reverb,
                                    srpgpu_stream_t stream) {
  SRPGPU_CHECK_ARG(num_samples >= 0 && num_mics >= 1 && num_images >= 1, SRPGPU_ERR_DIMENSION,
                   "render_images: bad shape (samples %lld, mics %d, images %d)", (long long)num_samples, num_mics,
                   num_images);
  SRPGPU_CHECK_ARG(dry && start && gain && taps && is_direct && direct && reverb, SRPGPU_ERR_VALUE,
                   "render_images: null buffer");
  const int64_t total = (int64_t)num_mics * num_samples;
  if (total == 0) return SRPGPU_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  rnd::render_images_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      dry, num_samples, num_mics, num_images, start, gain, taps, is_direct, direct, reverb);
  SRPGPU_CHECK_LAUNCH("render_images");
  return SRPGPU_OK;
}
