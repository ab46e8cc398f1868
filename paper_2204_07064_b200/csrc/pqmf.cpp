// pqmf.cpp — pseudo-QMF (cosine-modulated) filter bank for the RAVE-style configs.
//
// NOT in the reference (PQMF appears nowhere in SPEC/PAPER/proj): this is
// the builder's definition, parity-unpinned.  Design (all in double, rounded once to fp32):
//   prototype h: `taps`-tap Kaiser-windowed sinc lowpass, beta for 100 dB stop-band
//     (beta = 0.1102 (A - 8.7)), cutoff wc chosen by golden-section search to minimise
//     max_{n != 0} |(h * h~)[2 M n]| (the Kaiser-window PQMF criterion: the prototype's
//     autocorrelation must vanish at multiples of 2M for near-perfect reconstruction);
//   analysis  h_k[n] = 2 h[n] cos((2k+1) pi/(2M) (n - (N-1)/2) + (-1)^k pi/4)
//   synthesis g_k[n] = 2 h[n] cos((2k+1) pi/(2M) (n - (N-1)/2) - (-1)^k pi/4)
// Expressed as reference-layout conv weights (see sc_pqmf_filters in the header):
//   analysis CONV  (1 -> M, K=N, stride M, pad (N-M, 0)):  w[k][0][j] = h_k[N-1-j]
//   synthesis CONVT(M -> 1, K=N, stride M, pad (N-1, 0)):  w[0][k][j] = M g_k[N-1-j]
#include <cmath>
#include <vector>

#include "runtime.hpp"

namespace scb {

namespace {

double bessel_i0(double x) {
  double sum = 1.0, term = 1.0;
  const double q = x * x / 4.0;
  for (int k = 1; k < 200; ++k) {
    term *= q / (static_cast<double>(k) * k);
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}

std::vector<double> kaiser_lowpass(int N, double wc, double beta) {
  std::vector<double> h(N);
  const double c = (N - 1) / 2.0;
  const double i0b = bessel_i0(beta);
  for (int n = 0; n < N; ++n) {
    const double t = n - c;
    const double r = (N > 1) ? 2.0 * n / (N - 1) - 1.0 : 0.0;
    const double win = bessel_i0(beta * std::sqrt(std::max(0.0, 1.0 - r * r))) / i0b;
    const double sinc = (t == 0.0) ? wc / M_PI : std::sin(wc * t) / (M_PI * t);
    h[n] = sinc * win;
  }
  return h;
}

double objective(int N, int M, double wc, double beta) {
  const std::vector<double> h = kaiser_lowpass(N, wc, beta);
  double worst = 0.0;
  for (int lag = 2 * M; lag < N; lag += 2 * M) {
    double g = 0.0;
    for (int n = 0; n + lag < N; ++n) g += h[n] * h[n + lag];
    worst = std::max(worst, std::fabs(g));
  }
  return worst;
}

}  // namespace

void pqmf_filters(int M, int N, float* analysis, float* synthesis, double* prototype) {
  if (M < 2 || N < 2 * M) fail(SC_ERR_INVALID_ARGUMENT, "pqmf: need bands >= 2 and taps >= 2*bands");
  const double atten = 100.0;
  const double beta = 0.1102 * (atten - 8.7);
  // golden-section search of the cutoff around pi/(2M)
  const double gr = (std::sqrt(5.0) - 1.0) / 2.0;
  double a = 0.5 * M_PI / (2 * M), b = 1.5 * M_PI / (2 * M);
  double c = b - gr * (b - a), d = a + gr * (b - a);
  double fc = objective(N, M, c, beta), fd = objective(N, M, d, beta);
  for (int it = 0; it < 80; ++it) {
    if (fc < fd) {
      b = d;
      d = c;
      fd = fc;
      c = b - gr * (b - a);
      fc = objective(N, M, c, beta);
    } else {
      a = c;
      c = d;
      fc = fd;
      d = a + gr * (b - a);
      fd = objective(N, M, d, beta);
    }
  }
  const double wc = 0.5 * (a + b);
  const std::vector<double> h = kaiser_lowpass(N, wc, beta);
  const double cen = (N - 1) / 2.0;
  for (int k = 0; k < M; ++k) {
    const double ph = ((k % 2) ? -1.0 : 1.0) * M_PI / 4.0;
    for (int n = 0; n < N; ++n) {
      const double arg = (2 * k + 1) * M_PI / (2.0 * M) * (n - cen);
      const double hk = 2.0 * h[n] * std::cos(arg + ph);
      const double gk = 2.0 * h[n] * std::cos(arg - ph);
      const int j = N - 1 - n;
      if (analysis) analysis[static_cast<size_t>(k) * N + j] = static_cast<float>(hk);
      if (synthesis) synthesis[static_cast<size_t>(k) * N + j] = static_cast<float>(M * gk);
    }
  }
  if (analysis)
    for (int k = 0; k < M; ++k) analysis[static_cast<size_t>(M) * N + k] = 0.f;  // bias
  if (synthesis) synthesis[static_cast<size_t>(M) * N] = 0.f;                    // bias
  if (prototype)
    for (int n = 0; n < N; ++n) prototype[n] = h[n];
}

}  // namespace scb
