// ref_shim.cpp — C entry points over the REFERENCE's own tensor_core (test infrastructure).
//
// Compiled by oracle/Makefile together with the unmodified reference source
// /root/reference/proj/src/kernels.cpp into oracle/_ref/libref_streamconv.so.  The reference
// has no C ABI; this shim only converts plain arrays to the reference's
// SignalTensor / Kernel (proj/include/streamconv/tensor.hpp:14-88), calls the reference
// function and copies the result out.  Used to pin oracle/oracle.cpp (bit-exact conv1d) and
// as the "reference" CPU baseline (bench.py --impl reference).

#include <cstdint>
#include <cstring>
#include <vector>

#include "streamconv/kernels.hpp"

using namespace streamconv;

namespace {
SignalTensor make_sig(const float* x, int C, int64_t L) {
  SignalTensor t = SignalTensor::zeros(C, L);
  if (L > 0) std::memcpy(t.data.data(), x, sizeof(float) * static_cast<size_t>(C) * L);
  return t;
}
thread_local std::string g_err;
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// kernels.hpp:11-14
void ref_set_parallel_kernels(int enabled) { set_parallel_kernels(enabled != 0); }
int ref_parallel_kernels_enabled(void) { return parallel_kernels_enabled() ? 1 : 0; }

// kernels.hpp:18
int64_t ref_conv_output_length(int64_t L, int K, int S, int d) {
  return conv_output_length(L, K, S, d);
}

// conv1d (kernels.hpp:24, kernels.cpp:73-104) with the oracle's conv_fn_t signature.
void ref_conv1d(const float* x, int M, int64_t L, const float* w, const float* b, int N, int K,
                int S, int d, float* y) {
  SignalTensor xs = make_sig(x, M, L);
  Kernel k;
  k.out_channels = N;
  k.in_channels = M;
  k.taps = K;
  k.weights.assign(w, w + static_cast<size_t>(N) * M * K);
  k.bias.assign(b, b + N);
  SignalTensor ys = conv1d(xs, k, S, d);
  std::memcpy(y, ys.data.data(), sizeof(float) * ys.data.size());
}

// conv1d_serial (kernels.hpp:26) — returns 0 or 1 + ErrCode ordinal.
int ref_conv1d_checked(const float* x, int M, int64_t L, const float* w, const float* b, int N,
                       int K, int S, int d, float* y, int serial) {
  try {
    SignalTensor xs = make_sig(x, M, L);
    Kernel k;
    k.out_channels = N;
    k.in_channels = M;
    k.taps = K;
    k.weights.assign(w, w + static_cast<size_t>(N) * M * K);
    k.bias.assign(b, b + N);
    SignalTensor ys = serial ? conv1d_serial(xs, k, S, d) : conv1d(xs, k, S, d);
    std::memcpy(y, ys.data.data(), sizeof(float) * ys.data.size());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  }
}

// pad_zeros (kernels.hpp:16)
int ref_pad_zeros(const float* x, int C, int64_t L, int64_t left, int64_t right, float* y) {
  try {
    SignalTensor ys = pad_zeros(make_sig(x, C, L), PaddingSpec{left, right});
    if (!ys.data.empty()) std::memcpy(y, ys.data.data(), sizeof(float) * ys.data.size());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  }
}

// zero_upsample (kernels.hpp:30)
int ref_zero_upsample(const float* x, int C, int64_t L, int factor, float* y) {
  try {
    SignalTensor ys = zero_upsample(make_sig(x, C, L), factor);
    if (!ys.data.empty()) std::memcpy(y, ys.data.data(), sizeof(float) * ys.data.size());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  }
}

// activation (kernels.hpp:32)
int ref_activation(const float* x, int64_t n, int kind, float alpha, float* y) {
  SignalTensor ys = activation(make_sig(x, 1, n), static_cast<Act>(kind), alpha);
  if (n > 0) std::memcpy(y, ys.data.data(), sizeof(float) * n);
  return 0;
}

}  // extern "C"
