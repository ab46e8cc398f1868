// ola.cu — SPEC baseline_ola on the GPU: the unmodified non-causal graph run
// offline on overlapping windowed chunks, the paper's comparison baseline (§3.3, Fig. 10).
//
// Every chunk of every stream is one independent "stream" of an offline program (lower_dag
// with offline = true: original pads, no causalize delays, zero state per call), so all chunks
// of a call run batched through the same fused kernels as the streaming path:
//   gather   x[s][c][i*hop + n]            -> chunk (s*nc + i) [c][n]          (ola_gather)
//   offline  chunk batch through the plan  -> chunk outputs [s*nc+i][c'][N*sink]
//   add      y[s][c'][t] = sum_i w[t - i*hop'] * out_i[c'][t - i*hop']        (ola_add)
// with the ratio-scaled window w of length N*sink (hann_window; the 25% flat-
// top decision) and hop' = hop*sink; the output is trimmed to the input length.
#include <cmath>
#include <map>
#include <memory>

#include "runtime.hpp"

namespace scb {

namespace {

__global__ void ola_gather_kernel(const float* __restrict__ x, int streams, int C, int64_t T, int nc,
                                  int64_t hop, int64_t N, float* __restrict__ chunks) {
  const int64_t total = static_cast<int64_t>(streams) * nc * C * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = e % N;
    const int64_t r = e / N;
    const int c = static_cast<int>(r % C);
    const int64_t sc = r / C;  // s * nc + i
    const int64_t i = sc % nc, s = sc / nc;
    chunks[e] = x[(s * C + c) * T + i * hop + n];
  }
}

__global__ void ola_add_kernel(const float* __restrict__ out, int streams, int C, int nc, int64_t No,
                               int64_t hop_o, const float* __restrict__ w, int64_t To, float* __restrict__ y) {
  const int64_t total = static_cast<int64_t>(streams) * C * To;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = e % To;
    const int64_t r = e / To;
    const int c = static_cast<int>(r % C);
    const int64_t s = r / C;
    // chunks i with i*hop_o <= t < i*hop_o + No, ascending i (fixed summation order)
    int64_t i0 = (t >= No) ? (t - No) / hop_o + 1 : 0;
    const int64_t i1 = t / hop_o < nc - 1 ? t / hop_o : nc - 1;
    float acc = 0.f;
    for (int64_t i = i0; i <= i1; ++i) {
      const int64_t n = t - i * hop_o;
      acc += w[n] * out[((s * nc + i) * C + c) * No + n];
    }
    y[e] = acc;
  }
}

int grid_for_ola(int64_t items) {
  int64_t g = (items + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

// SPEC hann_window and the 25% flat-top decision, length Nw.
std::vector<double> ola_window(int64_t Nw, int overlap_pct) {
  std::vector<double> w(static_cast<size_t>(Nw), 1.0);
  const double pi = 3.14159265358979323846;
  if (overlap_pct == 50) {
    for (int64_t n = 0; n < Nw; ++n) {
      const double v = std::sin(pi * static_cast<double>(n) / static_cast<double>(Nw));
      w[n] = v * v;
    }
  } else if (overlap_pct == 25) {
    const int64_t q = Nw / 4;  // rising sin^2 quarter lobe, flat middle, falling quarter lobe
    for (int64_t n = 0; n < q; ++n) {
      const double v = std::sin(pi * static_cast<double>(n) / static_cast<double>(2 * q));
      w[n] = v * v;
      w[Nw - 1 - n] = std::sin(pi * static_cast<double>(n + 1) / static_cast<double>(2 * q)) *
                      std::sin(pi * static_cast<double>(n + 1) / static_cast<double>(2 * q));
    }
  }
  return w;
}

Ola::~Ola() {
  states.clear();
  if (plan && plan->device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(plan->device);
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_w);
    cudaSetDevice(prev);
  }
}

std::unique_ptr<Ola> make_ola(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
                              int64_t nW, int in_C, int precision, int device, int64_t chunk, int overlap_pct,
                              int streams, int64_t max_frames) {
  if (overlap_pct != 0 && overlap_pct != 25 && overlap_pct != 50)
    fail(SC_ERR_INVALID_ARGUMENT, "overlap must be 0, 25 or 50 (%)");
  if (precision != SC_PREC_FP32 && precision != SC_PREC_BF16)
    fail(SC_ERR_INVALID_ARGUMENT, "precision must be SC_PREC_FP32 or SC_PREC_BF16");
  if (streams < 1 || chunk < 1) fail(SC_ERR_INVALID_ARGUMENT, "streams and chunk must be >= 1");
  auto o = std::make_unique<Ola>();
  o->plan = make_plan(lower_dag(nodes, n, edges, ne, W, nW, in_C, true), precision, device);
  const Program& pg = o->plan->prog;
  if (chunk < pg.ratio)
    fail(SC_ERR_CHUNK_TOO_SMALL, "chunk " + std::to_string(chunk) + " is below the graph granularity " +
                                     std::to_string(pg.ratio));
  const int64_t hop = chunk * (100 - overlap_pct) / 100;
  if (chunk * (100 - overlap_pct) % 100 != 0 || hop % pg.ratio != 0 || chunk % pg.ratio != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "chunk and hop (" + std::to_string(hop) +
                                                  ") must be multiples of the compression ratio " +
                                                  std::to_string(pg.ratio));
  if ((chunk * pg.sink_rate.num) % pg.sink_rate.den || (hop * pg.sink_rate.num) % pg.sink_rate.den)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "chunk x sink rate is not an integer");
  if (max_frames < chunk) fail(SC_ERR_CHUNK_TOO_SMALL, "max_frames is shorter than one chunk");
  o->streams = streams;
  o->N = chunk;
  o->hop = hop;
  o->overlap = overlap_pct;
  o->max_frames = max_frames;
  if (device < 0) return o;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  const int64_t nc = (max_frames - chunk) / hop + 1;
  const int64_t No = chunk * pg.sink_rate.num / pg.sink_rate.den;
  o->in_floats = static_cast<int64_t>(streams) * nc * pg.in_C * chunk;
  o->out_floats = static_cast<int64_t>(streams) * nc * pg.sink_C * No;
  cudaError_t e = cudaMalloc(&o->d_in, o->in_floats * 4);
  if (e == cudaSuccess) e = cudaMalloc(&o->d_out, o->out_floats * 4);
  std::vector<double> wd = ola_window(No, overlap_pct);
  std::vector<float> wf(wd.begin(), wd.end());
  if (e == cudaSuccess) e = cudaMalloc(&o->d_w, wf.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(o->d_w, wf.data(), wf.size() * 4, cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) fail(SC_ERR_CUDA_BASE + static_cast<int>(e), std::string("OLA buffers: ") + cudaGetErrorString(e));
  return o;
}

const Plan& ola_plan(const Ola& o) { return *o.plan; }

void ola_process(Ola& o, const float* in, float* out, int64_t T, cudaStream_t s) {
  const Program& pg = o.plan->prog;
  if (o.plan->device < 0) fail(SC_ERR_INVALID_ARGUMENT, "OLA was created host-only (device -1)");
  if (T < o.N) fail(SC_ERR_CHUNK_TOO_SMALL, "signal shorter than one chunk");
  if (T % o.hop != 0) fail(SC_ERR_LENGTH_NOT_MULTIPLE_OF_RATIO, "signal length must be a multiple of the hop");
  if (T > o.max_frames) fail(SC_ERR_INVALID_ARGUMENT, "signal longer than max_frames");
  const int64_t nc = (T - o.N) / o.hop + 1;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(o.plan->device);
  auto it = o.states.find(nc);
  if (it == o.states.end())
    it = o.states.emplace(nc, make_state(o.plan.get(), static_cast<int>(o.streams * nc), o.N)).first;
  State& st = *it->second;
  const int64_t No = o.N * pg.sink_rate.num / pg.sink_rate.den;
  const int64_t hop_o = o.hop * pg.sink_rate.num / pg.sink_rate.den;
  const int64_t To = T * pg.sink_rate.num / pg.sink_rate.den;
  const int64_t gi = static_cast<int64_t>(o.streams) * nc * pg.in_C * o.N;
  ola_gather_kernel<<<grid_for_ola(gi), 256, 0, s>>>(in, o.streams, pg.in_C, T, static_cast<int>(nc), o.hop, o.N,
                                                     o.d_in);
  st.reset(nullptr, 0, s);  // every chunk starts from zero padding (offline_run)
  st.process(o.d_in, o.d_out, o.N, s);
  const int64_t ga = static_cast<int64_t>(o.streams) * pg.sink_C * To;
  ola_add_kernel<<<grid_for_ola(ga), 256, 0, s>>>(o.d_out, o.streams, pg.sink_C, static_cast<int>(nc), No, hop_o,
                                                  o.d_w, To, out);
  const cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  if (e != cudaSuccess) fail(SC_ERR_CUDA_BASE + static_cast<int>(e), std::string("OLA: ") + cudaGetErrorString(e));
}

}  // namespace scb
