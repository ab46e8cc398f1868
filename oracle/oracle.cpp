// oracle.cpp — CPU ORACLE (test infrastructure only; never on the product path).
//
// A plain restatement of the reference's algorithm for the north-star hot path, used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs as the
// checker.  Nothing under paper_2204_07064_b200/ links or calls this file.
//
// What it restates (each function cites the reference lines it follows):
//   - tensor_core: conv1d / pad_zeros / zero_upsample / activation / conv_output_length
//     (proj/src/kernels.cpp:36-128): fp32 storage, double accumulation per output in
//     m-then-k order, one cast to float per output.
//   - causalize: right->left pad rewrite, Eq. (2) stride delays inserted
//     as Delay nodes before strided convs, branch-alignment Delays at Sum, delay ledger.
//   - stream_runtime: per-stream StreamState with per-Conv caches of the
//     trailing L_total input samples and per-Delay rings, process_buffer, offline_run.
// The conv used by the executor is pluggable: the oracle's own restatement, or the
// reference's compiled conv1d from oracle/_ref (see oracle/ref_shim.cpp) for pinning and
// for the "reference" CPU baseline.
//
// Parity status: conv / strided conv / ConvT (zero_upsample + conv) /
// LeakyReLU / tanh / Delay+Sum are pinned by the reference code (oracle/_ref) and the SPEC
// known answers.  The GATE and SLICE nodes and the PQMF filter values have no reference; the
// oracle defines them, so their GPU parity is "unpinned" (checked against this oracle only).

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/streamconv_b200.h"

extern "C" int64_t oc_delay_for_stride(int64_t S, int64_t R, int64_t Dc);

namespace {

// ---------------------------------------------------------------- tensor_core restatement
// SignalTensor (tensor.hpp:14-48): channel-major [C][T] fp32.
struct Sig {
  int C = 1;
  int64_t T = 0;
  std::vector<float> d;
  Sig() = default;
  Sig(int c, int64_t t) : C(c), T(t), d(static_cast<size_t>(c) * static_cast<size_t>(t), 0.0f) {}
  float* ch(int c) { return d.data() + static_cast<size_t>(c) * T; }
  const float* ch(int c) const { return d.data() + static_cast<size_t>(c) * T; }
};

struct OracleError : std::runtime_error {
  int code;
  OracleError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_err;

// conv_output_length — kernels.cpp:46-49
int64_t out_len(int64_t L, int K, int S, int d) {
  const int64_t span = static_cast<int64_t>(K - 1) * d + 1;
  return (L - span) / S + 1;
}

// conv1d_serial — kernels.cpp:51-71 (the parallel path, kernels.cpp:73-104, is bit-identical
// by construction: same per-output accumulation order).
// x: [M][L], w: [N][M][K], b: [N], y: [N][Lout]
void conv1d_c(const float* x, int M, int64_t L, const float* w, const float* b, int N, int K,
              int S, int d, float* y) {
  const int64_t Lo = out_len(L, K, S, d);
  for (int n = 0; n < N; ++n) {
    float* yrow = y + static_cast<size_t>(n) * Lo;
    for (int64_t i = 0; i < Lo; ++i) {
      double acc = b[n];
      const int64_t base = i * S;
      for (int m = 0; m < M; ++m) {
        const float* xrow = x + static_cast<size_t>(m) * L;
        const float* wrow = w + (static_cast<size_t>(n) * M + m) * K;
        for (int t = 0; t < K; ++t)
          acc += static_cast<double>(wrow[t]) * xrow[base + static_cast<int64_t>(t) * d];
      }
      yrow[i] = static_cast<float>(acc);
    }
  }
}

typedef void (*conv_fn_t)(const float*, int, int64_t, const float*, const float*, int, int, int,
                          int, float*);

Sig conv(conv_fn_t fn, const Sig& x, int N, int K, int S, int d, const float* w, const float* b) {
  // check_conv_args — kernels.cpp:17-29
  const int64_t span = static_cast<int64_t>(K - 1) * d + 1;
  if (span > x.T) throw OracleError(SC_ERR_INPUT_TOO_SHORT, "conv1d input shorter than span");
  Sig y(N, out_len(x.T, K, S, d));
  fn(x.d.data(), x.C, x.T, w, b, N, K, S, d, y.d.data());
  return y;
}

// pad_zeros — kernels.cpp:36-44
Sig pad_zeros(const Sig& x, int64_t L, int64_t R) {
  Sig y(x.C, x.T + L + R);
  for (int c = 0; c < x.C; ++c) std::memcpy(y.ch(c) + L, x.ch(c), sizeof(float) * x.T);
  return y;
}

// zero_upsample — kernels.cpp:106-117
Sig zero_upsample(const Sig& x, int f) {
  if (f == 1) return x;
  Sig y(x.C, x.T * f);
  for (int c = 0; c < x.C; ++c)
    for (int64_t i = 0; i < x.T; ++i) y.ch(c)[i * f] = x.ch(c)[i];
  return y;
}

// activation — kernels.cpp:119-128
void activation_inplace(Sig& x, int kind, float alpha) {
  if (kind == SC_ACT_IDENTITY) return;
  if (kind == SC_ACT_TANH) {
    for (float& v : x.d) v = std::tanh(v);
  } else {
    for (float& v : x.d) v = v < 0.0f ? alpha * v : v;
  }
}

Sig concat_time(const Sig& a, const Sig& b) {
  Sig y(a.C, a.T + b.T);
  for (int c = 0; c < a.C; ++c) {
    std::memcpy(y.ch(c), a.ch(c), sizeof(float) * a.T);
    std::memcpy(y.ch(c) + a.T, b.ch(c), sizeof(float) * b.T);
  }
  return y;
}

Sig slice_time(const Sig& x, int64_t t0, int64_t n) {
  Sig y(x.C, n);
  for (int c = 0; c < x.C; ++c) std::memcpy(y.ch(c), x.ch(c) + t0, sizeof(float) * n);
  return y;
}

// ---------------------------------------------------------------- causalized program
enum OpKind { OP_CONV, OP_DELAY, OP_ZUP, OP_ACT, OP_GATE, OP_SLICE, OP_RES };

struct Prog;
struct Op {
  OpKind kind;
  int M = 0, N = 0, K = 1, S = 1, d = 1;
  int64_t L = 0, R = 0;      // original padding
  int64_t P = 0;             // causal left pad (L+R)
  const float* w = nullptr;
  const float* b = nullptr;
  int C = 0;                 // DELAY channels
  int64_t delay = 0;         // DELAY length (native-rate samples)
  int factor = 1;            // ZUP
  int act = 0;
  float alpha = 0.f;
  int sb = 0, sc = 0;        // SLICE
  std::shared_ptr<Prog> branch;  // RES
  int64_t skip_delay = 0;
  int skip_C = 0;
  int state = -1;            // index into per-stream state vector
  bool inserted = false;     // Delay inserted by causalize (not in the original graph)
};
struct Prog {
  std::vector<Op> ops;
};

struct Rate {
  int64_t num = 1, den = 1;
  void norm() {
    int64_t g = std::gcd(num, den);
    num /= g;
    den /= g;
  }
};

struct Graph {
  Prog root;
  int n_state = 0;
  int in_C = 1, out_C = 1;
  Rate sink;
  int64_t ratio = 1;
  int64_t latency_sink = 0;  // D_c at the sink (native rate)
  int64_t state_bytes = 0;   // SPEC.md:259 closed form (per stream)
  std::vector<int> state_C;  // channels of each state slot
  std::vector<int64_t> state_len;
};

struct Builder {
  const sc_node* nodes;
  int n;
  const float* W;
  int64_t nW;
  Graph* g;
  int pos = 0;

  int64_t lcm_acc = 1;

  int new_state(int C, int64_t len) {
    g->state_C.push_back(C);
    g->state_len.push_back(len);
    g->state_bytes += static_cast<int64_t>(C) * len * 4;
    return g->n_state++;
  }

  // Parse + causalize a sequence until RES_END (depth>0) or end.  C/D/rate are in/out.
  void parse(Prog& prog, int& C, int64_t& D, Rate& rate, int depth) {
    while (pos < n) {
      const sc_node& nd = nodes[pos];
      if (nd.kind == SC_NODE_RES_END) {
        if (depth == 0) throw OracleError(SC_ERR_MALFORMED_GRAPH, "RES_END without RES_BEGIN");
        return;
      }
      ++pos;
      switch (nd.kind) {
        case SC_NODE_CONV:
        case SC_NODE_CONVT: {
          if (nd.in_channels != C)
            throw OracleError(SC_ERR_CHANNEL_MISMATCH, "conv input channel mismatch");
          if (nd.in_channels < 1 || nd.out_channels < 1 || nd.taps < 1 || nd.stride < 1 ||
              nd.dilation < 1 || nd.pad_left < 0 || nd.pad_right < 0)
            throw OracleError(SC_ERR_INVALID_ARGUMENT, "conv shape");
          const int64_t need = static_cast<int64_t>(nd.out_channels) * nd.in_channels * nd.taps +
                               nd.out_channels;
          if (nd.weight_offset < 0 || nd.weight_offset + need > nW)
            throw OracleError(SC_ERR_INVALID_ARGUMENT, "weights out of range");
          Op op;
          op.kind = OP_CONV;
          op.M = nd.in_channels;
          op.N = nd.out_channels;
          op.K = nd.taps;
          op.L = nd.pad_left;
          op.R = nd.pad_right;
          op.P = nd.pad_left + nd.pad_right;
          op.w = W + nd.weight_offset;
          op.b = op.w + static_cast<int64_t>(nd.out_channels) * nd.in_channels * nd.taps;
          const int64_t span = static_cast<int64_t>(nd.taps - 1) * nd.dilation + 1;
          if (nd.kind == SC_NODE_CONVT) {
            if (nd.dilation != 1) throw OracleError(SC_ERR_INVALID_ARGUMENT, "convT dilation");
            if (op.P != nd.taps - 1)
              throw OracleError(SC_ERR_PADDING_NOT_STREAMABLE, "convT pad must total K-1");
            Op z;
            z.kind = OP_ZUP;
            z.factor = nd.stride;
            prog.ops.push_back(z);
            // ledger: ZeroUpsample D -> D*s
            D *= nd.stride;
            rate.num *= nd.stride;
            rate.norm();
            op.S = 1;
            op.d = 1;
          } else {
            op.S = nd.stride;
            op.d = nd.dilation;
            if (nd.stride == 1) {
              if (op.P != span - 1)
                throw OracleError(SC_ERR_PADDING_NOT_STREAMABLE, "pad must total (K-1)*d");
            } else {
              if (op.P < span - nd.stride)
                throw OracleError(SC_ERR_PADDING_NOT_STREAMABLE, "strided pad < span - S");
              // Eq. (2): D_a = (S - ((R + D_c) mod S)) mod S, Delay inserted before the
              // conv.
              const int64_t Da = oc_delay_for_stride(nd.stride, nd.pad_right, D);
              if (Da > 0) {
                Op dl;
                dl.kind = OP_DELAY;
                dl.C = C;
                dl.delay = Da;
                dl.inserted = true;
                dl.state = new_state(C, Da);
                prog.ops.push_back(dl);
              }
              if ((D + nd.pad_right + Da) % nd.stride != 0)
                throw OracleError(SC_ERR_INTERNAL_NON_INTEGER_DELAY, "ledger division");
              // ledger: strided conv D -> (D + R + D_a)/S
              D = (D + nd.pad_right + Da) / nd.stride;
              rate.den *= nd.stride;
              rate.norm();
            }
          }
          // ledger: pad (L,R)->(L+R,0) delays a stride-1 conv output by R
          if (nd.kind == SC_NODE_CONVT || nd.stride == 1) D += nd.pad_right;
          op.state = new_state(op.M, op.P);
          prog.ops.push_back(op);
          C = nd.out_channels;
          lcm_acc = std::lcm(lcm_acc, rate.den);
          break;
        }
        case SC_NODE_ACT: {
          if (nd.act < 0 || nd.act > 2) throw OracleError(SC_ERR_INVALID_ARGUMENT, "act kind");
          Op op;
          op.kind = OP_ACT;
          op.act = nd.act;
          op.alpha = nd.alpha;
          prog.ops.push_back(op);
          break;
        }
        case SC_NODE_GATE: {
          if (C % 2) throw OracleError(SC_ERR_CHANNEL_MISMATCH, "gate needs even channels");
          Op op;
          op.kind = OP_GATE;
          prog.ops.push_back(op);
          C /= 2;
          break;
        }
        case SC_NODE_SLICE: {
          if (nd.slice_begin < 0 || nd.slice_count < 1 || nd.slice_begin + nd.slice_count > C)
            throw OracleError(SC_ERR_CHANNEL_MISMATCH, "slice out of range");
          Op op;
          op.kind = OP_SLICE;
          op.sb = nd.slice_begin;
          op.sc = nd.slice_count;
          prog.ops.push_back(op);
          C = nd.slice_count;
          break;
        }
        case SC_NODE_RES_BEGIN: {
          Op op;
          op.kind = OP_RES;
          op.branch = std::make_shared<Prog>();
          int bC = C;
          int64_t bD = D;
          Rate br = rate;
          parse(*op.branch, bC, bD, br, depth + 1);
          if (pos >= n || nodes[pos].kind != SC_NODE_RES_END)
            throw OracleError(SC_ERR_MALFORMED_GRAPH, "RES_BEGIN without RES_END");
          ++pos;
          if (bC != C) throw OracleError(SC_ERR_CHANNEL_MISMATCH, "residual channels differ");
          if (br.num != rate.num || br.den != rate.den)
            throw OracleError(SC_ERR_RATE_MISMATCH_AT_SUM, "residual rates differ");
          // branch_alignment: A_i = max_j D_j - D_i
          const int64_t Dmax = std::max(bD, D);
          if (Dmax - bD != 0)
            throw OracleError(SC_ERR_MALFORMED_GRAPH, "branch needs delay (unsupported)");
          op.skip_delay = Dmax - D;
          op.skip_C = C;
          if (op.skip_delay > 0) op.state = new_state(C, op.skip_delay);
          prog.ops.push_back(op);
          D = Dmax;
          break;
        }
        default:
          throw OracleError(SC_ERR_SCHEMA_ERROR, "unknown node kind");
      }
    }
    if (depth > 0) throw OracleError(SC_ERR_MALFORMED_GRAPH, "RES_BEGIN without RES_END");
  }
};

void build_graph(const sc_node* nodes, int n, const float* W, int64_t nW, int in_C, Graph& g) {
  Builder b{nodes, n, W, nW, &g};
  int C = in_C;
  int64_t D = 0;
  Rate rate;
  g.in_C = in_C;
  b.parse(g.root, C, D, rate, 0);
  g.out_C = C;
  g.sink = rate;
  g.ratio = b.lcm_acc;
  g.latency_sink = D;
}

// ---------------------------------------------------------------- execution
struct StreamState {
  std::vector<Sig> slot;      // per state index: cache [C][len]
  std::vector<int64_t> n_in;  // per state index: input frames received (strided convs)
};

void init_state(const Graph& g, StreamState& st) {
  st.slot.clear();
  for (int i = 0; i < g.n_state; ++i) st.slot.emplace_back(g.state_C[i], g.state_len[i]);
  st.n_in.assign(g.n_state, 0);
}

// Delay(d): streaming = ring of d samples; offline = zero-prepend + truncate
Sig run_delay(const Sig& x, int64_t dly, Sig* ring) {
  if (dly == 0) return x;
  if (ring) {
    Sig xin = concat_time(*ring, x);
    Sig y = slice_time(xin, 0, x.T);
    *ring = slice_time(xin, xin.T - dly, dly);
    return y;
  }
  Sig z(x.C, dly);
  Sig xin = concat_time(z, x);
  return slice_time(xin, 0, x.T);
}

enum Mode { STREAM, OFFLINE_CAUSAL, OFFLINE_ORIGINAL };

Sig run_prog(const Prog& prog, Sig x, StreamState* st, Mode mode, conv_fn_t fn) {
  for (const Op& op : prog.ops) {
    switch (op.kind) {
      case OP_CONV: {
        const int64_t T = x.T;
        int64_t Tout = T / op.S;
        Sig xin;
        if (mode == STREAM) {
          // cached padding: xin = concat(cache, buf); the cache keeps the trailing input
          // samples the next output window starts at.  For a
          // stride-S conv fed buffers that are not multiples of S (phase state, buffers below
          // the compression ratio) the cache also holds the n_in mod S pending samples.
          Sig& cache = st->slot[op.state];
          const int64_t n_prev = st->n_in[op.state];
          const int64_t n_now = n_prev + T;
          Tout = n_now / op.S - n_prev / op.S;
          st->n_in[op.state] = n_now;
          xin = concat_time(cache, x);
          const int64_t keep = op.P + (n_now % op.S);
          cache = slice_time(xin, xin.T - keep, keep);
          if (Tout == 0) {
            x = Sig(op.N, 0);
            break;
          }
        } else if (mode == OFFLINE_CAUSAL) {
          xin = pad_zeros(x, op.P, 0);  // causalized pad (L+R, 0)
        } else {
          xin = pad_zeros(x, op.L, op.R);  // original pad
        }
        Sig y = conv(fn, xin, op.N, op.K, op.S, op.d, op.w, op.b);
        if (y.T < Tout) throw OracleError(SC_ERR_INPUT_TOO_SHORT, "conv produced too few");
        x = (y.T == Tout) ? std::move(y) : slice_time(y, 0, Tout);
        break;
      }
      case OP_DELAY:
        if (mode == OFFLINE_ORIGINAL) break;  // causalize-inserted: absent originally
        x = run_delay(x, op.delay, mode == STREAM ? &st->slot[op.state] : nullptr);
        break;
      case OP_ZUP:
        x = zero_upsample(x, op.factor);
        break;
      case OP_ACT:
        activation_inplace(x, op.act, op.alpha);
        break;
      case OP_GATE: {
        const int H = x.C / 2;
        Sig y(H, x.T);
        for (int c = 0; c < H; ++c)
          for (int64_t t = 0; t < x.T; ++t) {
            const float a = x.ch(c)[t];
            const float g = x.ch(c + H)[t];
            y.ch(c)[t] = std::tanh(a) * (1.0f / (1.0f + std::exp(-g)));
          }
        x = std::move(y);
        break;
      }
      case OP_SLICE: {
        Sig y(op.sc, x.T);
        for (int c = 0; c < op.sc; ++c)
          std::memcpy(y.ch(c), x.ch(op.sb + c), sizeof(float) * x.T);
        x = std::move(y);
        break;
      }
      case OP_RES: {
        Sig br = run_prog(*op.branch, x, st, mode, fn);
        Sig skip = (mode == OFFLINE_ORIGINAL)
                       ? x
                       : run_delay(x, op.skip_delay,
                                   (mode == STREAM && op.skip_delay > 0) ? &st->slot[op.state]
                                                                         : nullptr);
        // Sum: edge order branch + skip
        for (size_t i = 0; i < br.d.size(); ++i) br.d[i] = br.d[i] + skip.d[i];
        x = std::move(br);
        break;
      }
    }
  }
  return x;
}

conv_fn_t g_default_conv = conv1d_c;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SC_OK;
  } catch (const OracleError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SC_ERR_INVALID_ARGUMENT;
  }
}

// ---------------------------------------------------------------- SPEC graph_ir DAGs
// A second, independent restatement for general DAGs: the graph is
// validated minimally (the product's sc_graph_validate is tested separately), causalized as a
// literal graph-to-graph rewrite — pads (L,R) -> (L+R,0), Delay(D_a) nodes before strided
// convs (Eq. 2), Delay(A_i) nodes on Sum inputs (branch_alignment) — and executed node by
// node in topological order: Conv caches / Delay rings per node in streaming mode
// (SPEC.md:255-280), zero-prepend + truncate offline.
struct DagG {
  std::vector<sc_gnode> nd;       // causalized nodes (original ids kept, inserted appended)
  std::vector<int64_t> L0, R0;    // original pads per node (OFFLINE_ORIGINAL)
  std::vector<sc_edge> ed;
  std::vector<std::vector<int>> in_e, out_e;
  std::vector<int> order;
  std::vector<int> slot;          // state slot per node (-1: none)
  std::vector<int> slot_C;
  std::vector<int64_t> slot_len;
  int in_C = 1, out_C = 1;
  Rate sink;
  int64_t ratio = 1, latency_in = 0, state_bytes = 0;
};

int d_inputs(const sc_gnode& g) { return g.kind == SC_G_SOURCE ? 0 : g.kind == SC_G_SUM ? g.arity : 1; }

void dag_topo(DagG& g) {
  const int n = static_cast<int>(g.nd.size());
  g.in_e.assign(n, {});
  g.out_e.assign(n, {});
  for (int i = 0; i < n; ++i) g.in_e[i].assign(d_inputs(g.nd[i]), -1);
  for (size_t e = 0; e < g.ed.size(); ++e) {
    const sc_edge& x = g.ed[e];
    if (x.from < 0 || x.from >= n || x.to < 0 || x.to >= n || x.port < 0 ||
        x.port >= static_cast<int>(g.in_e[x.to].size()) || g.in_e[x.to][x.port] >= 0)
      throw OracleError(SC_ERR_MALFORMED_GRAPH, "bad edge");
    g.in_e[x.to][x.port] = static_cast<int>(e);
    g.out_e[x.from].push_back(static_cast<int>(e));
  }
  std::vector<int> done(n, 0);
  g.order.clear();
  for (bool progress = true; progress;) {
    progress = false;
    for (int i = 0; i < n; ++i) {
      if (done[i]) continue;
      bool ready = true;
      for (int e : g.in_e[i]) ready = ready && e >= 0 && done[g.ed[e].from];
      if (ready) {
        done[i] = 1;
        g.order.push_back(i);
        progress = true;
      }
    }
  }
  if (static_cast<int>(g.order.size()) != n) throw OracleError(SC_ERR_CYCLE_DETECTED, "cycle");
}

void dag_build(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
               int64_t nW, int in_C, DagG& g) {
  (void)W;  // weights are read by dag_pass; here only their ranges are checked
  g.nd.assign(nodes, nodes + n);
  g.ed.assign(edges, edges + ne);
  g.in_C = in_C;
  dag_topo(g);
  // rates, channels and the ledger on the ORIGINAL graph
  std::vector<int> C(ne, 0);
  std::vector<Rate> rate(ne);
  std::vector<int64_t> D(ne, 0), ins(ne, 0);
  for (int u : g.order) {
    const sc_gnode& x = g.nd[u];
    int c = in_C;
    Rate r;
    int64_t d = 0;
    if (x.kind != SC_G_SOURCE) {
      const int e0 = g.in_e[u][0];
      c = C[e0];
      r = rate[e0];
      d = D[e0];
    }
    switch (x.kind) {
      case SC_G_CONV: {
        if (x.in_channels != c) throw OracleError(SC_ERR_CHANNEL_MISMATCH, "conv channels");
        const int64_t need = static_cast<int64_t>(x.out_channels) * x.in_channels * x.taps + x.out_channels;
        if (x.weight_offset < 0 || x.weight_offset + need > nW) throw OracleError(SC_ERR_INVALID_ARGUMENT, "weights");
        const int64_t R = x.pad_right + x.shift;
        const int64_t span = static_cast<int64_t>(x.taps - 1) * x.dilation + 1;
        const int64_t P = x.pad_left + x.pad_right;
        if (x.stride == 1 ? P != span - 1 : P < span - x.stride)
          throw OracleError(SC_ERR_PADDING_NOT_STREAMABLE, "conv padding");
        if (x.stride > 1) {
          const int64_t Da = oc_delay_for_stride(x.stride, R, d);  // Eq. (2)
          ins[g.in_e[u][0]] = Da;
          d = (d + R + Da) / x.stride;
          r.den *= x.stride;
        } else {
          d += R;
        }
        c = x.out_channels;
        break;
      }
      case SC_G_ZERO_UPSAMPLE:
        d *= x.factor;
        r.num *= x.factor;
        break;
      case SC_G_DELAY:
        if (x.inserted) d += x.samples;  // a model Delay shifts original and causal alike
        break;
      case SC_G_SUM: {
        for (int q = 0; q < x.arity; ++q) {
          const int e = g.in_e[u][q];
          if (C[e] != c) throw OracleError(SC_ERR_CHANNEL_MISMATCH, "sum channels");
          if (rate[e].num * r.den != r.num * rate[e].den) throw OracleError(SC_ERR_RATE_MISMATCH_AT_SUM, "sum rates");
          d = std::max(d, D[e]);
        }
        for (int q = 0; q < x.arity; ++q) ins[g.in_e[u][q]] = d - D[g.in_e[u][q]];  // A_i
        break;
      }
      case SC_G_GATE:
        c /= 2;
        break;
      case SC_G_SLICE:
        if (x.slice_begin < 0 || x.slice_count < 1 || x.slice_begin + x.slice_count > c)
          throw OracleError(SC_ERR_CHANNEL_MISMATCH, "slice");
        c = x.slice_count;
        break;
      case SC_G_SINK:
        g.out_C = c;
        g.sink = r;
        g.latency_in = d * r.den / r.num;
        break;
      default:
        break;
    }
    r.norm();
    for (int e : g.out_e[u]) {
      C[e] = c;
      rate[e] = r;
      D[e] = d;
      g.ratio = std::lcm(g.ratio, r.den);
    }
  }
  // the causalize rewrite: inserted Delay nodes on their edges, causal pads
  g.L0.assign(n, 0);
  g.R0.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    sc_gnode& x = g.nd[i];
    g.L0[i] = x.pad_left;
    g.R0[i] = x.pad_right;
    if (x.kind == SC_G_CONV) {
      x.pad_left += x.pad_right;
      x.pad_right = 0;
    }
  }
  std::vector<sc_edge> ed2;
  for (int e = 0; e < ne; ++e) {
    if (ins[e] == 0) {
      ed2.push_back(g.ed[e]);
      continue;
    }
    sc_gnode dl{};
    dl.kind = SC_G_DELAY;
    dl.samples = ins[e];
    dl.inserted = 1;
    dl.in_channels = C[e];
    const int id = static_cast<int>(g.nd.size());
    g.nd.push_back(dl);
    g.L0.push_back(0);
    g.R0.push_back(0);
    ed2.push_back(sc_edge{g.ed[e].from, id, 0});
    ed2.push_back(sc_edge{id, g.ed[e].to, g.ed[e].port});
  }
  g.ed.swap(ed2);
  dag_topo(g);
  // state slots: conv caches (causal pad at the conv's input rate), Delay rings
  std::vector<int> C2(g.ed.size(), 0);
  g.slot.assign(g.nd.size(), -1);
  for (int u : g.order) {
    const sc_gnode& x = g.nd[u];
    int c = x.kind == SC_G_SOURCE ? in_C : C2[g.in_e[u][0]];
    int64_t len = 0;
    if (x.kind == SC_G_CONV) {
      len = x.pad_left;
      g.slot[u] = static_cast<int>(g.slot_C.size());
      g.slot_C.push_back(c);
      g.slot_len.push_back(len);
      c = x.out_channels;
    } else if (x.kind == SC_G_DELAY) {
      len = x.samples;
      g.slot[u] = static_cast<int>(g.slot_C.size());
      g.slot_C.push_back(c);
      g.slot_len.push_back(len);
    } else if (x.kind == SC_G_GATE) {
      c /= 2;
    } else if (x.kind == SC_G_SLICE) {
      c = x.slice_count;
    }
    if (g.slot[u] >= 0) g.state_bytes += static_cast<int64_t>(g.slot_C[g.slot[u]]) * len * 4;
    for (int e : g.out_e[u]) C2[e] = c;
  }
}

// One pass of the DAG over a buffer (STREAM) or a whole signal (offline modes).
Sig dag_pass(const DagG& g, const float* W, Sig x, StreamState* st, Mode mode, conv_fn_t fn) {
  std::vector<Sig> val(g.ed.size());
  Sig out;
  for (int u : g.order) {
    const sc_gnode& nd = g.nd[u];
    Sig v;
    if (nd.kind == SC_G_SOURCE) {
      v = std::move(x);
    } else if (nd.kind != SC_G_SUM) {
      v = val[g.in_e[u][0]];
    }
    switch (nd.kind) {
      case SC_G_CONV: {
        const float* w = W + nd.weight_offset;
        const float* b = w + static_cast<int64_t>(nd.out_channels) * nd.in_channels * nd.taps;
        const int S = nd.stride;
        int64_t Tout = v.T / S;
        Sig xin;
        if (mode == STREAM) {
          Sig& cache = st->slot[g.slot[u]];
          const int64_t n_prev = st->n_in[g.slot[u]];
          const int64_t n_now = n_prev + v.T;
          Tout = n_now / S - n_prev / S;
          st->n_in[g.slot[u]] = n_now;
          xin = concat_time(cache, v);
          const int64_t keep = nd.pad_left + (n_now % S);
          cache = slice_time(xin, xin.T - keep, keep);
          if (Tout == 0) {
            v = Sig(nd.out_channels, 0);
            break;
          }
        } else if (mode == OFFLINE_CAUSAL) {
          xin = pad_zeros(v, nd.pad_left, 0);
        } else {
          xin = pad_zeros(v, g.L0[u], g.R0[u]);
        }
        Sig y = conv(fn, xin, nd.out_channels, nd.taps, S, nd.dilation, w, b);
        if (y.T < Tout) throw OracleError(SC_ERR_INPUT_TOO_SHORT, "conv produced too few");
        v = (y.T == Tout) ? std::move(y) : slice_time(y, 0, Tout);
        break;
      }
      case SC_G_ZERO_UPSAMPLE:
        v = zero_upsample(v, nd.factor);
        break;
      case SC_G_ACTIVATION:
        activation_inplace(v, nd.act, nd.alpha);
        break;
      case SC_G_DELAY:
        if (mode == OFFLINE_ORIGINAL && nd.inserted) break;  // absent from the original graph
        v = run_delay(v, nd.samples, (mode == STREAM && nd.samples > 0) ? &st->slot[g.slot[u]] : nullptr);
        break;
      case SC_G_SUM: {
        v = val[g.in_e[u][0]];
        for (int q = 1; q < nd.arity; ++q) {
          const Sig& o = val[g.in_e[u][q]];
          if (o.T != v.T || o.C != v.C) throw OracleError(SC_ERR_LENGTH_MISMATCH, "sum operands differ in length");
          for (size_t i = 0; i < v.d.size(); ++i) v.d[i] = v.d[i] + o.d[i];  // port order
        }
        break;
      }
      case SC_G_GATE: {
        const int H = v.C / 2;
        Sig y(H, v.T);
        for (int c = 0; c < H; ++c)
          for (int64_t t = 0; t < v.T; ++t)
            y.ch(c)[t] = std::tanh(v.ch(c)[t]) * (1.0f / (1.0f + std::exp(-v.ch(c + H)[t])));
        v = std::move(y);
        break;
      }
      case SC_G_SLICE: {
        Sig y(nd.slice_count, v.T);
        for (int c = 0; c < nd.slice_count; ++c) std::memcpy(y.ch(c), v.ch(nd.slice_begin + c), sizeof(float) * v.T);
        v = std::move(y);
        break;
      }
      case SC_G_SINK:
        out = v;
        break;
      default:
        break;
    }
    for (int e : g.out_e[u]) val[e] = v;
  }
  return out;
}

}  // namespace

extern "C" {

// DAG versions of oc_graph_info / oc_run (same conventions, sc_gnode / sc_edge graphs).
int oc_dag_info(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
                int64_t nW, int in_C, int64_t* info) {
  return guard([&] {
    DagG g;
    dag_build(nodes, n, edges, ne, W, nW, in_C, g);
    info[0] = g.ratio;
    info[1] = g.sink.num;
    info[2] = g.sink.den;
    info[3] = g.out_C;
    info[4] = g.latency_in;
    info[5] = g.state_bytes;
  });
}

int oc_dag_run(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
               int64_t nW, int in_C, int n_streams, const float* x, int64_t T_total,
               const int64_t* parts, int n_parts, float* y, int mode, void* conv_fn, int threads) {
  return guard([&] {
    DagG g;
    dag_build(nodes, n, edges, ne, W, nW, in_C, g);
    conv_fn_t fn = conv_fn ? reinterpret_cast<conv_fn_t>(conv_fn) : g_default_conv;
    const bool phase = mode == 3;
    if (phase) mode = 0;
    int64_t sum = 0;
    for (int p = 0; p < n_parts; ++p) {
      if (parts[p] <= 0 || (!phase && parts[p] % g.ratio != 0))
        throw OracleError(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "buffer not multiple of ratio");
      sum += parts[p];
    }
    if (mode != 0 && T_total % g.ratio != 0)
      throw OracleError(SC_ERR_LENGTH_NOT_MULTIPLE_OF_RATIO, "length not multiple of ratio");
    if (mode == 0 && sum != T_total) throw OracleError(SC_ERR_LENGTH_MISMATCH, "parts do not sum to length");
    const int64_t Tout_total = T_total * g.sink.num / g.sink.den;
    std::vector<std::string> errs(n_streams);
    std::vector<int> codes(n_streams, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int s = 0; s < n_streams; ++s) {
      try {
        const float* xs = x + static_cast<size_t>(s) * in_C * T_total;
        float* ys = y + static_cast<size_t>(s) * g.out_C * Tout_total;
        if (mode == 0) {
          StreamState st;
          for (size_t k = 0; k < g.slot_C.size(); ++k) st.slot.emplace_back(g.slot_C[k], g.slot_len[k]);
          st.n_in.assign(g.slot_C.size(), 0);
          int64_t t0 = 0, o0 = 0;
          for (int p = 0; p < n_parts; ++p) {
            Sig buf(in_C, parts[p]);
            for (int c = 0; c < in_C; ++c)
              std::memcpy(buf.ch(c), xs + static_cast<size_t>(c) * T_total + t0, sizeof(float) * parts[p]);
            Sig out = dag_pass(g, W, std::move(buf), &st, STREAM, fn);
            for (int c = 0; c < g.out_C; ++c)
              std::memcpy(ys + static_cast<size_t>(c) * Tout_total + o0, out.ch(c), sizeof(float) * out.T);
            t0 += parts[p];
            o0 += out.T;
          }
        } else {
          Sig buf(in_C, T_total);
          std::memcpy(buf.d.data(), xs, sizeof(float) * in_C * T_total);
          Sig out = dag_pass(g, W, std::move(buf), nullptr, mode == 1 ? OFFLINE_CAUSAL : OFFLINE_ORIGINAL, fn);
          if (out.T != Tout_total) throw OracleError(SC_ERR_LENGTH_MISMATCH, "sink length");
          std::memcpy(ys, out.d.data(), sizeof(float) * out.d.size());
        }
      } catch (const OracleError& e) {
        errs[s] = e.what();
        codes[s] = e.code;
      }
    }
    for (int s = 0; s < n_streams; ++s)
      if (codes[s]) throw OracleError(codes[s], errs[s]);
  });
}

}  // extern "C"

extern "C" {

// delay_for_stride, Eq. (2)
int64_t oc_delay_for_stride(int64_t S, int64_t R, int64_t Dc) { return (S - ((R + Dc) % S)) % S; }

const char* oc_last_error(void) { return g_err.c_str(); }

int64_t oc_conv_output_length(int64_t L, int K, int S, int d) { return out_len(L, K, S, d); }

void oc_conv1d(const float* x, int M, int64_t L, const float* w, const float* b, int N, int K,
               int S, int d, float* y) {
  conv1d_c(x, M, L, w, b, N, K, S, d, y);
}

// NOT a restatement: a deliberately fp32-ACCUMULATING conv with the same signature, used only
// as evidence for the RES_SCALE decision (configs.py, tests/test_oracle.py): how large is the
// error of ANY fp32-accumulating implementation against the reference's double accumulation
// (kernels.cpp:96-100)?  "BLAS order": the (m, k) reduction of each output is split over 8
// interleaved fp32 partial sums (one SIMD register's worth), combined pairwise at the end.
// `sequential` != 0: one fp32 accumulator in the reference's m-then-k order instead.
static int g_f32_sequential = 0;
void oc_set_f32acc_order(int sequential) { g_f32_sequential = sequential; }
void oc_conv1d_f32acc(const float* x, int M, int64_t L, const float* w, const float* b, int N,
                      int K, int S, int d, float* y) {
  const int64_t Lo = out_len(L, K, S, d);
  for (int n = 0; n < N; ++n)
    for (int64_t i = 0; i < Lo; ++i) {
      float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int64_t j = 0;
      for (int m = 0; m < M; ++m) {
        const float* xrow = x + static_cast<size_t>(m) * L + i * S;
        const float* wrow = w + (static_cast<size_t>(n) * M + m) * K;
        for (int t = 0; t < K; ++t, ++j) {
          const float p = wrow[t] * xrow[static_cast<int64_t>(t) * d];
          if (g_f32_sequential) part[0] += p; else part[j & 7] += p;
        }
      }
      const float s4[4] = {part[0] + part[4], part[1] + part[5], part[2] + part[6], part[3] + part[7]};
      y[static_cast<size_t>(n) * Lo + i] = b[n] + ((s4[0] + s4[2]) + (s4[1] + s4[3]));
    }
}

int oc_branch_alignment(const int64_t* D, int n, int64_t* A) {
  // SPEC.md:200-204
  if (n < 1) return SC_ERR_INVALID_ARGUMENT;
  int64_t mx = D[0];
  for (int i = 1; i < n; ++i) mx = std::max(mx, D[i]);
  for (int i = 0; i < n; ++i) A[i] = mx - D[i];
  return SC_OK;
}

void oc_pad_zeros(const float* x, int C, int64_t T, int64_t L, int64_t R, float* y) {
  Sig s(C, T);
  std::memcpy(s.d.data(), x, sizeof(float) * C * T);
  Sig o = pad_zeros(s, L, R);
  std::memcpy(y, o.d.data(), sizeof(float) * o.d.size());
}

void oc_zero_upsample(const float* x, int C, int64_t T, int f, float* y) {
  Sig s(C, T);
  std::memcpy(s.d.data(), x, sizeof(float) * C * T);
  Sig o = zero_upsample(s, f);
  std::memcpy(y, o.d.data(), sizeof(float) * o.d.size());
}

void oc_activation(const float* x, int64_t n, int kind, float alpha, float* y) {
  Sig s(1, n);
  std::memcpy(s.d.data(), x, sizeof(float) * n);
  activation_inplace(s, kind, alpha);
  std::memcpy(y, s.d.data(), sizeof(float) * n);
}

// Graph facts after causalize: [ratio, sink_num, sink_den, out_C, latency_sink, state_bytes]
int oc_graph_info(const sc_node* nodes, int n, const float* W, int64_t nW, int in_C,
                  int64_t* info) {
  return guard([&] {
    Graph g;
    build_graph(nodes, n, W, nW, in_C, g);
    info[0] = g.ratio;
    info[1] = g.sink.num;
    info[2] = g.sink.den;
    info[3] = g.out_C;
    info[4] = g.latency_sink;
    info[5] = g.state_bytes;
  });
}

// Streaming run (process_buffer) for `n_streams` independent streams.
// x: [n_streams][in_C][T_total]; the per-stream signal is cut into consecutive buffers of
// lengths `parts[0..n_parts)` (sum = T_total, each a multiple of the ratio) and the outputs
// concatenated into y: [n_streams][out_C][T_total*sink].  mode: 0 stream, 1 offline of the
// causalized graph (offline_run), 2 offline of the ORIGINAL graph, 3 stream
// with phase state: buffers need not be multiples of the compression ratio; every node emits
// what its accumulated input allows and the per-call outputs are concatenated (the sink then
// lags the input by up to ratio - buffer samples; the GPU emits the same stream delayed by a
// fixed D, see sc_process).
// conv_fn: NULL = oracle restatement; else a kernels.cpp-compatible conv (oracle/_ref).
// threads: OpenMP threads across streams (SPEC.md:302,304 allow independent states to run
// concurrently); 0 = runtime default.
int oc_run(const sc_node* nodes, int n, const float* W, int64_t nW, int in_C, int n_streams,
           const float* x, int64_t T_total, const int64_t* parts, int n_parts, float* y,
           int mode, void* conv_fn, int threads) {
  return guard([&] {
    Graph g;
    build_graph(nodes, n, W, nW, in_C, g);
    conv_fn_t fn = conv_fn ? reinterpret_cast<conv_fn_t>(conv_fn) : g_default_conv;
    int64_t sum = 0;
    const bool phase = mode == 3;
    if (phase) mode = 0;
    for (int p = 0; p < n_parts; ++p) {
      if (parts[p] <= 0 || (!phase && parts[p] % g.ratio != 0))
        throw OracleError(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "buffer not multiple of ratio");
      if (phase && (parts[p] * g.sink.num) % g.sink.den != 0)
        throw OracleError(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "buffer x sink rate not integral");
      sum += parts[p];
    }
    if (mode != 0) {
      if (T_total % g.ratio != 0)
        throw OracleError(SC_ERR_LENGTH_NOT_MULTIPLE_OF_RATIO, "length not multiple of ratio");
    } else if (sum != T_total) {
      throw OracleError(SC_ERR_LENGTH_MISMATCH, "parts do not sum to length");
    }
    const int64_t Tout_total = T_total * g.sink.num / g.sink.den;
    std::vector<std::string> errs(n_streams);
    std::vector<int> codes(n_streams, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int s = 0; s < n_streams; ++s) {
      try {
        const float* xs = x + static_cast<size_t>(s) * in_C * T_total;
        float* ys = y + static_cast<size_t>(s) * g.out_C * Tout_total;
        if (mode == 0) {
          StreamState st;
          init_state(g, st);  // zero-initialized caches
          int64_t t0 = 0, o0 = 0;
          for (int p = 0; p < n_parts; ++p) {
            Sig buf(in_C, parts[p]);
            for (int c = 0; c < in_C; ++c)
              std::memcpy(buf.ch(c), xs + static_cast<size_t>(c) * T_total + t0,
                          sizeof(float) * parts[p]);
            Sig out = run_prog(g.root, std::move(buf), &st, STREAM, fn);
            for (int c = 0; c < g.out_C; ++c)
              std::memcpy(ys + static_cast<size_t>(c) * Tout_total + o0, out.ch(c),
                          sizeof(float) * out.T);
            t0 += parts[p];
            o0 += out.T;
          }
        } else {
          Sig buf(in_C, T_total);
          std::memcpy(buf.d.data(), xs, sizeof(float) * in_C * T_total);
          Sig out = run_prog(g.root, std::move(buf), nullptr,
                             mode == 1 ? OFFLINE_CAUSAL : OFFLINE_ORIGINAL, fn);
          std::memcpy(ys, out.d.data(), sizeof(float) * out.d.size());
        }
      } catch (const OracleError& e) {
        errs[s] = e.what();
        codes[s] = e.code;
      }
    }
    for (int s = 0; s < n_streams; ++s)
      if (codes[s]) throw OracleError(codes[s], errs[s]);
  });
}

}  // extern "C"
