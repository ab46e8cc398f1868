// C++ cached-module API test (include/streamconv_b200.hpp over the C-ABI).
//   test_modules host   : plan facts + typed errors (no GPU)
//   test_modules gpu    : stream a small residual stack, partition bit-identity, reset
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "streamconv_b200.hpp"

using namespace streamconv::b200;

static std::vector<float> lcg(size_t n, uint32_t seed, float scale) {
  std::vector<float> v(n);
  uint32_t s = seed;
  for (auto& x : v) {
    s = s * 1664525u + 1013904223u;
    x = scale * (static_cast<float>(s >> 8) / 16777216.0f * 2.0f - 1.0f);
  }
  return v;
}

static Sequential model() {
  Sequential m(16);
  for (int d : {1, 3}) {
    m.residual([&](Sequential& br) {
      br.leaky_relu(0.2f);
      br.conv(CachedConv1d{16, 16, 3, 1, d, {d, d}, lcg(16 * 16 * 3, 7 + d, 0.25f), {}});
      br.leaky_relu(0.2f);
      br.conv(CachedConv1d{16, 16, 1, 1, 1, {0, 0}, lcg(16 * 16, 11 + d, 0.4f), lcg(16, 3, 0.1f)});
    });
  }
  return m;
}

#define REQUIRE(c)                                              \
  do {                                                          \
    if (!(c)) {                                                 \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                 \
    }                                                           \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  Sequential m = model();
  {
    Plan host(m, -1);
    REQUIRE(host.ratio() == 1);
    REQUIRE(host.latency() == 4);                     // centered K=3: d=1 + d=3
    REQUIRE(host.state_bytes() == 16 * 4 * 3 * 4);    // sum_d (2d conv cache + d skip) x 16 ch x 4 B
    bool threw = false;
    try {
      Sequential bad(8);
      bad.conv(CachedConv1d{16, 16, 3});
      Plan p(bad, -1);
    } catch (const Error& e) {
      threw = e.code() == "ChannelMismatch";
    }
    REQUIRE(threw);
  }
  {
    // SPEC graph_ir DAG: a centered residual unit with a 3-way Sum and a model Delay
    Graph g(4);
    const int x = g.source();
    const int a = g.conv(x, CachedConv1d{4, 4, 3, 1, 1, {1, 1}, lcg(48, 5, 0.3f), {}});
    const int b = g.conv(g.leaky_relu(x, 0.2f), CachedConv1d{4, 4, 5, 1, 1, {2, 2}, lcg(80, 6, 0.3f), {}});
    g.sink(g.sum({a, b, g.delay(x, 1)}));
    int64_t past = 0, future = 0;
    g.receptive_field(&past, &future);
    REQUIRE(past == 2 && future == 2);
    REQUIRE(g.compression_ratio() == 1);
    REQUIRE(g.causalize_latency() == 2);
    bool nc = false;
    try {
      g.latency();
    } catch (const Error& e) {
      nc = e.code() == "NotCausal";
    }
    REQUIRE(nc);
    Plan hp(g, -1);
    REQUIRE(hp.latency() == 2);
    g.save("/tmp/sc_cpp_model.json");
    Model m2("/tmp/sc_cpp_model.json");
    REQUIRE(m2.n_nodes() == 8 && m2.in_channels() == 4);  // 7 + the Fanout of x
    Plan hp2(m2, -1);
    REQUIRE(hp2.latency() == 2 && hp2.state_bytes() == hp.state_bytes());
  }
  if (!gpu) {
    std::printf("OK host\n");
    return 0;
  }
  const int S = 3, C = 16, T = 512;
  Plan plan(m, 0);
  StreamBatch st(plan, S, T);
  std::vector<float> x = lcg(static_cast<size_t>(S) * C * T, 99, 1.0f);
  float *dx, *dy1, *dy2;
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&dy1, x.size() * 4);
  cudaMalloc(&dy2, x.size() * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  st.process_buffer(dx, dy1, T);
  // same signal as two halves: [S][C][T/2] slices must be contiguous per call
  std::vector<float> a(static_cast<size_t>(S) * C * T / 2), b(a.size());
  for (int s = 0; s < S; ++s)
    for (int c = 0; c < C; ++c) {
      std::memcpy(&a[(static_cast<size_t>(s) * C + c) * T / 2], &x[(static_cast<size_t>(s) * C + c) * T], 4 * T / 2);
      std::memcpy(&b[(static_cast<size_t>(s) * C + c) * T / 2], &x[(static_cast<size_t>(s) * C + c) * T + T / 2], 4 * T / 2);
    }
  float *da, *db, *ya, *yb;
  cudaMalloc(&da, a.size() * 4);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&ya, a.size() * 4);
  cudaMalloc(&yb, b.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  st.reset();
  st.process_buffer(da, ya, T / 2);
  st.process_buffer(db, yb, T / 2);
  cudaDeviceSynchronize();
  std::vector<float> y1(x.size()), h1(a.size()), h2(b.size());
  cudaMemcpy(y1.data(), dy1, y1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h1.data(), ya, h1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), yb, h2.size() * 4, cudaMemcpyDeviceToHost);
  double rms = 0;
  for (float v : y1) rms += static_cast<double>(v) * v;
  REQUIRE(rms > 0);
  for (int s = 0; s < S; ++s)
    for (int c = 0; c < C; ++c) {
      const float* full = &y1[(static_cast<size_t>(s) * C + c) * T];
      REQUIRE(std::memcmp(full, &h1[(static_cast<size_t>(s) * C + c) * T / 2], 4 * T / 2) == 0);
      REQUIRE(std::memcmp(full + T / 2, &h2[(static_cast<size_t>(s) * C + c) * T / 2], 4 * T / 2) == 0);
    }
  bool threw = false;
  try {
    st.process_buffer(dx, dy1, 2 * T);  // > max_frames
  } catch (const Error& e) {
    threw = e.code() == "InvalidArgument";
  }
  REQUIRE(threw);
  {
    // the DAG through the GPU: one buffer vs two halves must be bit-identical, and the OLA
    // baseline over the same graph runs
    Graph g(C);
    const int x0 = g.source();
    const int a0 = g.conv(x0, CachedConv1d{C, C, 3, 1, 1, {1, 1}, lcg(C * C * 3, 5, 0.2f), {}});
    const int b0 = g.conv(g.leaky_relu(x0, 0.2f), CachedConv1d{C, C, 5, 1, 1, {2, 2}, lcg(C * C * 5, 6, 0.2f), {}});
    g.sink(g.sum({a0, b0, g.delay(x0, 1)}));
    Plan gp(g, 0);
    StreamBatch gs(gp, S, T);
    gs.process_buffer(dx, dy1, T);
    gs.reset();
    gs.process_buffer(da, ya, T / 2);
    gs.process_buffer(db, yb, T / 2);
    cudaDeviceSynchronize();
    cudaMemcpy(y1.data(), dy1, y1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1.data(), ya, h1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), yb, h2.size() * 4, cudaMemcpyDeviceToHost);
    for (int s = 0; s < S; ++s)
      for (int c = 0; c < C; ++c) {
        const float* full = &y1[(static_cast<size_t>(s) * C + c) * T];
        REQUIRE(std::memcmp(full, &h1[(static_cast<size_t>(s) * C + c) * T / 2], 4 * T / 2) == 0);
        REQUIRE(std::memcmp(full + T / 2, &h2[(static_cast<size_t>(s) * C + c) * T / 2], 4 * T / 2) == 0);
      }
    OverlapAdd ola(g, 128, 50, S, T);
    ola.process(dx, dy2, T);
    REQUIRE(cudaDeviceSynchronize() == cudaSuccess);
  }
  std::printf("OK gpu\n");
  return 0;
}
