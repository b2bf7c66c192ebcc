// esi_metrics.cu -- frame-vs-ground-truth scores (SPEC
// metrics S:401-437): per frame, the Pearson correlation of the 8-bit frame with
// the ground-truth log-intensity field and the mean squared error after
// per-image zero-mean, unit-variance normalisation (SPEC FrameScore S:406).
// Both are invariant to positive-affine rescaling, which is the paper's
// "relative intensity instead of absolute values" claim (Sec. III-A).
//
// One CTA per frame; the five moment sums are accumulated in fp64 (the frame
// holds up to ~4 M pixels).  With n pixels, means mx, my and
//   sxx = S(x - mx)^2, syy = S(y - my)^2, sxy = S(x - mx)(y - my):
//   pearson = sxy / sqrt(sxx syy),   mse_norm = mean((zx - zy)^2) = 2 (1 - pearson)
// (z = (v - m) / sqrt(s / n), population standard deviation).  Either image
// constant: both scores are NaN ("missing").
#include "esi_device.cuh"

namespace esi {

__global__ void __launch_bounds__(512) esi_frame_metrics_kernel(const uint8_t* frames, const float* truth,
                                                                int64_t P, int truth_per_frame, double* pearson,
                                                                double* mse_norm) {
  const int j = blockIdx.x;
  const uint8_t* f = frames + (int64_t)j * P;
  const float* g = truth + (truth_per_frame ? (int64_t)j * P : 0);
  // two passes (means, then centred moments) for fp64 accuracy without cancellation
  __shared__ double red[5][16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double sx = 0, sy = 0;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
    sx += (double)f[i];
    sy += (double)g[i];
  }
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(kFull, sx, o);
    sy += __shfl_xor_sync(kFull, sy, o);
  }
  if (lane == 0) { red[0][warp] = sx; red[1][warp] = sy; }
  __syncthreads();
  double mx = 0, my = 0;
  for (int w = 0; w < nw; ++w) { mx += red[0][w]; my += red[1][w]; }
  mx /= (double)P;
  my /= (double)P;
  __syncthreads();
  double sxx = 0, syy = 0, sxy = 0;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
    const double dx = (double)f[i] - mx, dy = (double)g[i] - my;
    sxx += dx * dx;
    syy += dy * dy;
    sxy += dx * dy;
  }
  for (int o = 16; o; o >>= 1) {
    sxx += __shfl_xor_sync(kFull, sxx, o);
    syy += __shfl_xor_sync(kFull, syy, o);
    sxy += __shfl_xor_sync(kFull, sxy, o);
  }
  if (lane == 0) { red[2][warp] = sxx; red[3][warp] = syy; red[4][warp] = sxy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int w = 0; w < nw; ++w) { a += red[2][w]; b += red[3][w]; c += red[4][w]; }
    if (a > 0.0 && b > 0.0) {
      const double r = c / sqrt(a * b);
      pearson[j] = r;
      mse_norm[j] = 2.0 * (1.0 - r);
    } else {
      pearson[j] = __longlong_as_double(0x7ff8000000000000ll);   // NaN: missing (constant image)
      mse_norm[j] = __longlong_as_double(0x7ff8000000000000ll);
    }
  }
}

cudaError_t launch_frame_metrics(const uint8_t* frames, const float* truth, int64_t P, int n_frames,
                                 int truth_per_frame, double* pearson, double* mse_norm, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  esi_frame_metrics_kernel<<<n_frames, 512, 0, s>>>(frames, truth, P, truth_per_frame, pearson, mse_norm);
  return cudaGetLastError();
}

}  // namespace esi
