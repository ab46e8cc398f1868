// metrics.cu — SPEC metrics_bench fidelity scores on batches of signals:
//   spectral_distance  L_s = sum over n_fft in {256, 512, 1024} (hop n_fft/4, Hann analysis
//                      window) of || log(|STFT x| + 1) - log(|STFT y| + 1) ||_2 / frames
//                      (Eq. 3, epsilon = 1; the scale set is SPEC's stated decision)
//   euclidean_distance L_w = || x - y ||_2                                        (Eq. 4)
//   correlation        L_c = sum x y / sqrt(sum x^2 sum y^2)                      (draft Eq.)
//   best_lag           argmax over lag in [0, max_lag] of correlation(ref[0:T-lag], test[lag:T])
// Reductions accumulate in double; the STFT is cuFFT (library FFT, like cuBLAS for GEMMs).
#include <cufft.h>

#include <cmath>
#include <vector>

#include "runtime.hpp"

namespace scb {

namespace {

void ckfft(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) fail(SC_ERR_CUDA_BASE + 999, std::string(what) + ": cuFFT error " + std::to_string(r));
}

// per signal: sum (x-y)^2, sum x y, sum x^2, sum y^2 (block per signal, double accumulation)
__global__ void moments_kernel(const float* __restrict__ x, const float* __restrict__ y, int64_t T,
                               double* __restrict__ out) {
  const int64_t s = blockIdx.x;
  const float* xs = x + s * T;
  const float* ys = y + s * T;
  double d2 = 0, xy = 0, xx = 0, yy = 0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const double a = xs[t], b = ys[t];
    d2 += (a - b) * (a - b);
    xy += a * b;
    xx += a * a;
    yy += b * b;
  }
  __shared__ double red[4][32];
  double v[4] = {d2, xy, xx, yy};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double a = threadIdx.x < (blockDim.x >> 5) ? red[k][threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) out[s * 4 + k] = a;
    }
  }
}

// windowed frames of signals [s0, s0 + ns): frames[(s * F + f) * n + k] = w[k] x[s][f*hop + k]
__global__ void frames_kernel(const float* __restrict__ x, int64_t T, int ns, int F, int n, int hop,
                              float* __restrict__ fr) {
  const int64_t total = static_cast<int64_t>(ns) * F * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e % n);
    const int64_t sf = e / n;
    const int f = static_cast<int>(sf % F);
    const int64_t s = sf / F;
    const float w = sinpif(static_cast<float>(k) / static_cast<float>(n));
    fr[e] = w * w * x[s * T + static_cast<int64_t>(f) * hop + k];
  }
}

// per signal: sum over frames and bins of (log(|X|+1) - log(|Y|+1))^2
__global__ void logspec_diff_kernel(const cufftComplex* __restrict__ X, const cufftComplex* __restrict__ Y,
                                    int64_t per_signal, double* __restrict__ out) {
  const int64_t s = blockIdx.x;
  double acc = 0;
  for (int64_t i = threadIdx.x; i < per_signal; i += blockDim.x) {
    const cufftComplex a = X[s * per_signal + i], b = Y[s * per_signal + i];
    const double la = log1p(sqrt(static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y));
    const double lb = log1p(sqrt(static_cast<double>(b.x) * b.x + static_cast<double>(b.y) * b.y));
    acc += (la - lb) * (la - lb);
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) out[s] += a;
  }
}

// lag-correlation sums for lags [0, L]: out[(s * (L+1) + lag) * 3] = (sum r t, sum r^2, sum t^2)
// over r = ref[0 : T-lag], t = test[lag : T]
__global__ void lag_kernel(const float* __restrict__ ref, const float* __restrict__ test, int64_t T, int L,
                           double* __restrict__ out) {
  const int lag = blockIdx.x;
  const int64_t s = blockIdx.y;
  const float* r = ref + s * T;
  const float* q = test + s * T + lag;
  double rt = 0, rr = 0, tt = 0;
  for (int64_t i = threadIdx.x; i < T - lag; i += blockDim.x) {
    const double a = r[i], b = q[i];
    rt += a * b;
    rr += a * a;
    tt += b * b;
  }
  __shared__ double red[3][32];
  double v[3] = {rt, rr, tt};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double a = threadIdx.x < (blockDim.x >> 5) ? red[k][threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) out[(s * (L + 1) + lag) * 3 + k] = a;
    }
  }
}

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SC_ERR_CUDA_BASE + static_cast<int>(e), std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// moments[n][4] = (sum (x-y)^2, sum x y, sum x^2, sum y^2), host doubles
void signal_moments(const float* x, const float* y, int n, int64_t T, double* moments, cudaStream_t st) {
  double* d = nullptr;
  ckc(cudaMallocAsync(&d, sizeof(double) * 4 * n, st), "cudaMallocAsync");
  moments_kernel<<<n, 256, 0, st>>>(x, y, T, d);
  ckc(cudaMemcpyAsync(moments, d, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  ckc(cudaFreeAsync(d, st), "cudaFreeAsync");
  ckc(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

void spectral_distance(const float* x, const float* y, int n, int64_t T, double* out, cudaStream_t st) {
  std::vector<double> acc(n, 0.0);
  for (int i = 0; i < n; ++i) out[i] = 0.0;
  for (int nfft : {256, 512, 1024}) {
    const int hop = nfft / 4;
    if (T < nfft) continue;  // no full frame at this scale
    const int64_t F64 = 1 + (T - nfft) / hop;
    const int F = static_cast<int>(F64);
    const int bins = nfft / 2 + 1;
    // signals per batch: keep the frame buffers near 256 MB
    const int64_t per = F64 * nfft * 4 * 2 + F64 * bins * 8 * 2;
    const int nb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n, (int64_t{256} << 20) / per)));
    float *fx = nullptr, *fy = nullptr;
    cufftComplex *X = nullptr, *Y = nullptr;
    double* d = nullptr;
    ckc(cudaMalloc(&fx, sizeof(float) * nb * F64 * nfft), "cudaMalloc");
    ckc(cudaMalloc(&fy, sizeof(float) * nb * F64 * nfft), "cudaMalloc");
    ckc(cudaMalloc(&X, sizeof(cufftComplex) * nb * F64 * bins), "cudaMalloc");
    ckc(cudaMalloc(&Y, sizeof(cufftComplex) * nb * F64 * bins), "cudaMalloc");
    ckc(cudaMalloc(&d, sizeof(double) * n), "cudaMalloc");
    ckc(cudaMemsetAsync(d, 0, sizeof(double) * n, st), "cudaMemsetAsync");
    cufftHandle plan;
    int dims[1] = {nfft};
    ckfft(cufftPlanMany(&plan, 1, dims, nullptr, 1, nfft, nullptr, 1, bins, CUFFT_R2C, nb * F), "cufftPlanMany");
    ckfft(cufftSetStream(plan, st), "cufftSetStream");
    for (int s0 = 0; s0 < n; s0 += nb) {
      const int ns = std::min(nb, n - s0);
      const int64_t items = static_cast<int64_t>(nb) * F * nfft;
      const int grid = static_cast<int>(std::min<int64_t>((items + 255) / 256, 148 * 16));
      if (ns < nb) {  // the plan is batched for nb signals: zero the unused tail
        ckc(cudaMemsetAsync(fx, 0, sizeof(float) * items, st), "memset");
        ckc(cudaMemsetAsync(fy, 0, sizeof(float) * items, st), "memset");
      }
      frames_kernel<<<grid, 256, 0, st>>>(x + static_cast<int64_t>(s0) * T, T, ns, F, nfft, hop, fx);
      frames_kernel<<<grid, 256, 0, st>>>(y + static_cast<int64_t>(s0) * T, T, ns, F, nfft, hop, fy);
      ckfft(cufftExecR2C(plan, fx, X), "cufftExecR2C");
      ckfft(cufftExecR2C(plan, fy, Y), "cufftExecR2C");
      logspec_diff_kernel<<<ns, 256, 0, st>>>(X, Y, F64 * bins, d + s0);
    }
    ckc(cudaMemcpyAsync(acc.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    ckc(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    cufftDestroy(plan);
    cudaFree(fx);
    cudaFree(fy);
    cudaFree(X);
    cudaFree(Y);
    cudaFree(d);
    for (int i = 0; i < n; ++i) out[i] += std::sqrt(acc[i]) / static_cast<double>(F);
  }
}

void best_lag(const float* ref, const float* test, int n, int64_t T, int max_lag, int64_t* lags, cudaStream_t st) {
  if (max_lag < 0 || max_lag >= T) fail(SC_ERR_INVALID_ARGUMENT, "max_lag must be in [0, T)");
  const int64_t cnt = static_cast<int64_t>(n) * (max_lag + 1) * 3;
  std::vector<double> h(static_cast<size_t>(cnt));
  double* d = nullptr;
  ckc(cudaMallocAsync(&d, sizeof(double) * cnt, st), "cudaMallocAsync");
  lag_kernel<<<dim3(max_lag + 1, n), 256, 0, st>>>(ref, test, T, max_lag, d);
  ckc(cudaMemcpyAsync(h.data(), d, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  ckc(cudaFreeAsync(d, st), "cudaFreeAsync");
  ckc(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  for (int s = 0; s < n; ++s) {
    int64_t best = -1;
    double bv = -2.0;
    for (int l = 0; l <= max_lag; ++l) {
      const double* v = &h[(static_cast<size_t>(s) * (max_lag + 1) + l) * 3];
      if (v[1] <= 0 || v[2] <= 0) continue;
      const double c = v[0] / std::sqrt(v[1] * v[2]);
      if (c > bv) bv = c, best = l;
    }
    if (best < 0) fail(SC_ERR_ZERO_ENERGY, "signal " + std::to_string(s) + " has zero energy at every lag");
    lags[s] = best;
  }
}

}  // namespace scb
