// streamconv_b200.hpp — C++ cached-module API over the C-ABI (header-only).
//
// The host-side mirror of the reference's streaming interface: cached modules (SPEC.md
// graph_ir node kinds) are appended to a Sequential stack, compiled into a
// Plan (causalize) and run for a batch of independent streams
// (stream_runtime).  Errors are rethrown as streamconv::b200::Error carrying
// the reference ErrCode name (error.hpp:8-70).
//
//   streamconv::b200::Sequential m(128);
//   m.residual([](auto& br) { br.leaky_relu(0.2f).conv(CachedConv1d{128, 128, 3, 1, 9}); });
//   streamconv::b200::Plan plan(m);                 // device 0
//   streamconv::b200::StreamBatch st(plan, 256, 2048);
//   st.process_buffer(d_in, d_out, 2048, stream);
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "streamconv_b200.h"

namespace streamconv {
namespace b200 {

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
  int status() const noexcept { return status_; }
  std::string code() const { return sc_status_name(status_); }  // e.g. "ChannelMismatch"

 private:
  int status_;
};

inline void check(int st) {
  if (st != SC_OK) throw Error(st, sc_last_error());
}

// ---- cached modules -------------------------------------------------------------------
// Padding: {-1, -1} selects the centered (non-causal, trained) padding; the plan causalizes.
struct PaddingSpec {
  int64_t left = -1, right = -1;
};

struct CachedConv1d {  // conv1d(pad(x,(L,R)), k, stride, dilation)   kernels.cpp:73-104
  int in_channels, out_channels, taps, stride = 1, dilation = 1;
  PaddingSpec padding{};
  std::vector<float> weights;  // [n][m][k] (tensor.hpp:52-88); empty = zeros
  std::vector<float> bias;     // [n]; empty = zeros
};

struct CachedConvTranspose1d {  // zero_upsample(stride) + conv1d
  int in_channels, out_channels, taps, stride;
  PaddingSpec padding{};
  std::vector<float> weights;  // conv-form kernel [n][m][k]
  std::vector<float> bias;
};

class Sequential {
 public:
  explicit Sequential(int in_channels) : in_channels_(in_channels), channels_(in_channels) {}

  int in_channels() const { return in_channels_; }
  int channels() const { return channels_; }
  const std::vector<sc_node>& nodes() const { return nodes_; }
  const std::vector<float>& weights() const { return weights_; }

  Sequential& conv(const CachedConv1d& c) {
    PaddingSpec p = c.padding;
    if (p.left < 0) {
      const int64_t tot = c.stride == 1 ? static_cast<int64_t>(c.taps - 1) * c.dilation : c.taps - 1;
      p = {(tot + 1) / 2, tot / 2};
    }
    sc_node n = base(SC_NODE_CONV);
    n.in_channels = c.in_channels;
    n.out_channels = c.out_channels;
    n.taps = c.taps;
    n.stride = c.stride;
    n.dilation = c.dilation;
    n.pad_left = p.left;
    n.pad_right = p.right;
    n.weight_offset = add_weights(c.weights, c.bias, c.out_channels, c.in_channels, c.taps);
    nodes_.push_back(n);
    channels_ = c.out_channels;
    return *this;
  }

  Sequential& conv_transpose(const CachedConvTranspose1d& c) {
    PaddingSpec p = c.padding;
    if (p.left < 0) p = {c.taps / 2, (c.taps - 1) / 2};
    sc_node n = base(SC_NODE_CONVT);
    n.in_channels = c.in_channels;
    n.out_channels = c.out_channels;
    n.taps = c.taps;
    n.stride = c.stride;
    n.pad_left = p.left;
    n.pad_right = p.right;
    n.weight_offset = add_weights(c.weights, c.bias, c.out_channels, c.in_channels, c.taps);
    nodes_.push_back(n);
    channels_ = c.out_channels;
    return *this;
  }

  // activation (kernels.cpp:119-128); the reference default alpha is 0.01f (kernels.hpp:32)
  Sequential& leaky_relu(float alpha = 0.01f) { return act(SC_ACT_LEAKY_RELU, alpha); }
  Sequential& tanh() { return act(SC_ACT_TANH, 0.f); }

  // Fanout -> branch -> Sum(branch, Delay_A(skip)), A from branch_alignment
  Sequential& residual(const std::function<void(Sequential&)>& branch) {
    nodes_.push_back(base(SC_NODE_RES_BEGIN));
    const int c0 = channels_;
    branch(*this);
    if (channels_ != c0) throw Error(SC_ERR_CHANNEL_MISMATCH, "ChannelMismatch: residual branch changes channels");
    nodes_.push_back(base(SC_NODE_RES_END));
    return *this;
  }

  Sequential& gate() {  // y = tanh(x[:C/2]) * sigmoid(x[C/2:])
    nodes_.push_back(base(SC_NODE_GATE));
    channels_ /= 2;
    return *this;
  }

  Sequential& slice(int begin, int count) {
    sc_node n = base(SC_NODE_SLICE);
    n.slice_begin = begin;
    n.slice_count = count;
    nodes_.push_back(n);
    channels_ = count;
    return *this;
  }

  // PQMF analysis / synthesis (builder-defined, sc_pqmf_filters)
  Sequential& pqmf_analysis(int bands = 16, int taps = 256) {
    std::vector<float> ana(static_cast<size_t>(bands) * taps + bands), syn(static_cast<size_t>(bands) * taps + 1);
    check(sc_pqmf_filters(bands, taps, ana.data(), syn.data(), nullptr));
    CachedConv1d c{1, bands, taps, bands, 1, {taps - bands, 0}, {}, {}};
    c.weights.assign(ana.begin(), ana.begin() + static_cast<size_t>(bands) * taps);
    c.bias.assign(bands, 0.f);
    conv(c);
    nodes_.back().hint = SC_HINT_PQMF;
    return *this;
  }
  Sequential& pqmf_synthesis(int bands = 16, int taps = 256) {
    std::vector<float> ana(static_cast<size_t>(bands) * taps + bands), syn(static_cast<size_t>(bands) * taps + 1);
    check(sc_pqmf_filters(bands, taps, ana.data(), syn.data(), nullptr));
    CachedConvTranspose1d c{bands, 1, taps, bands, {taps - 1, 0}, {}, {}};
    c.weights.assign(syn.begin(), syn.begin() + static_cast<size_t>(bands) * taps);
    c.bias.assign(1, 0.f);
    conv_transpose(c);
    nodes_.back().hint = SC_HINT_PQMF;
    return *this;
  }

 private:
  static sc_node base(int kind) {
    sc_node n{};
    n.kind = kind;
    n.stride = 1;
    n.dilation = 1;
    return n;
  }
  Sequential& act(int kind, float alpha) {
    sc_node n = base(SC_NODE_ACT);
    n.act = kind;
    n.alpha = alpha;
    nodes_.push_back(n);
    return *this;
  }
  int64_t add_weights(const std::vector<float>& w, const std::vector<float>& b, int N, int M, int K) {
    const int64_t off = static_cast<int64_t>(weights_.size());
    const size_t nw = static_cast<size_t>(N) * M * K;
    if (!w.empty() && w.size() != nw)
      throw Error(SC_ERR_INVALID_ARGUMENT, "InvalidArgument: kernel weight count does not match shape");
    if (!b.empty() && b.size() != static_cast<size_t>(N))
      throw Error(SC_ERR_INVALID_ARGUMENT, "InvalidArgument: kernel bias count does not match out_channels");
    if (w.empty()) weights_.resize(weights_.size() + nw, 0.f); else weights_.insert(weights_.end(), w.begin(), w.end());
    if (b.empty()) weights_.resize(weights_.size() + N, 0.f); else weights_.insert(weights_.end(), b.begin(), b.end());
    return off;
  }

  int in_channels_, channels_;
  std::vector<sc_node> nodes_;
  std::vector<float> weights_;
};

// ---- SPEC graph_ir DAG ------------------------------------------------
// Builder methods take the producing node id(s) and return the new node's id; a node feeding
// several consumers gets its Fanout inserted by finalize() (SPEC houses branching in Fanout).
class Graph {
 public:
  explicit Graph(int in_channels) : in_channels_(in_channels) {
    sc_gnode n = base(SC_G_SOURCE);
    n.out_channels = in_channels;
    source_ = push(n, {});
  }

  int in_channels() const { return in_channels_; }
  int source() const { return source_; }

  int conv(int x, const CachedConv1d& c) {
    PaddingSpec p = c.padding;
    if (p.left < 0) {
      const int64_t tot = c.stride == 1 ? static_cast<int64_t>(c.taps - 1) * c.dilation : c.taps - 1;
      p = {(tot + 1) / 2, tot / 2};
    }
    sc_gnode n = base(SC_G_CONV);
    n.in_channels = c.in_channels;
    n.out_channels = c.out_channels;
    n.taps = c.taps;
    n.stride = c.stride;
    n.dilation = c.dilation;
    n.pad_left = p.left;
    n.pad_right = p.right;
    n.weight_offset = add_weights(c.weights, c.bias, c.out_channels, c.in_channels, c.taps);
    return push(n, {x});
  }
  int zero_upsample(int x, int factor) {
    sc_gnode n = base(SC_G_ZERO_UPSAMPLE);
    n.factor = factor;
    return push(n, {x});
  }
  int leaky_relu(int x, float alpha = 0.01f) { return act(x, SC_ACT_LEAKY_RELU, alpha); }
  int tanh(int x) { return act(x, SC_ACT_TANH, 0.f); }
  int delay(int x, int64_t samples) {
    sc_gnode n = base(SC_G_DELAY);
    n.samples = samples;
    return push(n, {x});
  }
  int sum(const std::vector<int>& xs) {
    sc_gnode n = base(SC_G_SUM);
    n.arity = static_cast<int32_t>(xs.size());
    return push(n, xs);
  }
  int gate(int x) { return push(base(SC_G_GATE), {x}); }
  int slice(int x, int begin, int count) {
    sc_gnode n = base(SC_G_SLICE);
    n.slice_begin = begin;
    n.slice_count = count;
    return push(n, {x});
  }
  int sink(int x) { return push(base(SC_G_SINK), {x}); }

  // the C-ABI arrays (Fanouts inserted, edge order kept: Sum operand order)
  void finalize(std::vector<sc_gnode>* nodes, std::vector<sc_edge>* edges) const {
    *nodes = nodes_;
    edges->clear();
    std::vector<int> uses(nodes_.size(), 0), fan(nodes_.size(), -1);
    for (const sc_edge& e : edges_) ++uses[e.from];
    for (size_t i = 0; i < nodes_.size(); ++i)
      if (uses[i] > 1 && nodes_[i].kind != SC_G_FANOUT) {
        sc_gnode f = base(SC_G_FANOUT);
        f.arity = uses[i];
        fan[i] = static_cast<int>(nodes->size());
        nodes->push_back(f);
      }
    for (const sc_edge& e : edges_) edges->push_back(sc_edge{fan[e.from] >= 0 ? fan[e.from] : e.from, e.to, e.port});
    for (size_t i = 0; i < nodes_.size(); ++i)
      if (fan[i] >= 0) edges->push_back(sc_edge{static_cast<int32_t>(i), fan[i], 0});
  }
  const std::vector<float>& weights() const { return weights_; }

  // SPEC analyses
  int64_t compression_ratio() const {
    Arrays a(*this);
    int64_t r = 0;
    check(sc_graph_compression_ratio(a.n.data(), a.nn(), a.e.data(), a.ne(), in_channels_, &r));
    return r;
  }
  void receptive_field(int64_t* past, int64_t* future) const {
    Arrays a(*this);
    check(sc_graph_receptive_field(a.n.data(), a.nn(), a.e.data(), a.ne(), in_channels_, past, future));
  }
  int64_t latency() const {  // latency_of: NotCausal when future context remains
    Arrays a(*this);
    int64_t r = 0;
    check(sc_graph_latency(a.n.data(), a.nn(), a.e.data(), a.ne(), in_channels_, &r));
    return r;
  }
  int64_t causalize_latency() const {
    Arrays a(*this);
    int64_t r = 0;
    check(sc_graph_causalize(a.n.data(), a.nn(), a.e.data(), a.ne(), in_channels_, nullptr, 0, nullptr, nullptr, 0,
                             nullptr, &r));
    return r;
  }
  // model_io
  void save(const std::string& manifest, const char* blob = nullptr) const {
    Arrays a(*this);
    check(sc_model_save(manifest.c_str(), blob, a.n.data(), a.nn(), a.e.data(), a.ne(), weights_.data(),
                        static_cast<int64_t>(weights_.size()), in_channels_));
  }

  struct Arrays {
    std::vector<sc_gnode> n;
    std::vector<sc_edge> e;
    explicit Arrays(const Graph& g) { g.finalize(&n, &e); }
    int32_t nn() const { return static_cast<int32_t>(n.size()); }
    int32_t ne() const { return static_cast<int32_t>(e.size()); }
  };

 private:
  static sc_gnode base(int kind) {
    sc_gnode n{};
    n.kind = kind;
    n.stride = 1;
    n.dilation = 1;
    n.factor = 1;
    return n;
  }
  int act(int x, int kind, float alpha) {
    sc_gnode n = base(SC_G_ACTIVATION);
    n.act = kind;
    n.alpha = alpha;
    return push(n, {x});
  }
  int push(const sc_gnode& n, const std::vector<int>& inputs) {
    const int id = static_cast<int>(nodes_.size());
    nodes_.push_back(n);
    for (size_t q = 0; q < inputs.size(); ++q) edges_.push_back(sc_edge{inputs[q], id, static_cast<int32_t>(q)});
    return id;
  }
  int64_t add_weights(const std::vector<float>& w, const std::vector<float>& b, int N, int M, int K) {
    const int64_t off = static_cast<int64_t>(weights_.size());
    const size_t nw = static_cast<size_t>(N) * M * K;
    if (!w.empty() && w.size() != nw)
      throw Error(SC_ERR_INVALID_ARGUMENT, "InvalidArgument: kernel weight count does not match shape");
    if (!b.empty() && b.size() != static_cast<size_t>(N))
      throw Error(SC_ERR_INVALID_ARGUMENT, "InvalidArgument: kernel bias count does not match out_channels");
    if (w.empty()) weights_.resize(weights_.size() + nw, 0.f); else weights_.insert(weights_.end(), w.begin(), w.end());
    if (b.empty()) weights_.resize(weights_.size() + N, 0.f); else weights_.insert(weights_.end(), b.begin(), b.end());
    return off;
  }

  int in_channels_;
  int source_ = 0;
  std::vector<sc_gnode> nodes_;
  std::vector<sc_edge> edges_;
  std::vector<float> weights_;
};

// A model loaded from a model_io manifest (JSON + f32 blob): arrays owned by the library.
class Model {
 public:
  explicit Model(const std::string& manifest, const char* blob = nullptr) {
    check(sc_model_load(manifest.c_str(), blob, &m_));
    check(sc_model_graph(m_, &nodes_, &n_nodes_, &edges_, &n_edges_, &weights_, &n_weights_, &in_channels_));
  }
  ~Model() { sc_model_destroy(m_); }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  const sc_gnode* nodes() const { return nodes_; }
  int32_t n_nodes() const { return n_nodes_; }
  const sc_edge* edges() const { return edges_; }
  int32_t n_edges() const { return n_edges_; }
  const float* weights() const { return weights_; }
  int64_t n_weights() const { return n_weights_; }
  int32_t in_channels() const { return in_channels_; }

 private:
  sc_model* m_ = nullptr;
  const sc_gnode* nodes_ = nullptr;
  const sc_edge* edges_ = nullptr;
  const float* weights_ = nullptr;
  int32_t n_nodes_ = 0, n_edges_ = 0, in_channels_ = 0;
  int64_t n_weights_ = 0;
};

// ---- plan + stream batch --------------------------------------------------------------
class Plan {
 public:
  explicit Plan(const Sequential& m, int device = 0, int precision = SC_PREC_FP32) {
    check(sc_plan_create(m.nodes().data(), static_cast<int32_t>(m.nodes().size()), m.weights().data(),
                         static_cast<int64_t>(m.weights().size()), m.in_channels(), precision, device, &p_));
  }
  explicit Plan(const Graph& g, int device = 0, int precision = SC_PREC_FP32) {
    Graph::Arrays a(g);
    check(sc_plan_create_graph(a.n.data(), a.nn(), a.e.data(), a.ne(), g.weights().data(),
                               static_cast<int64_t>(g.weights().size()), g.in_channels(), precision, device, &p_));
  }
  explicit Plan(const Model& m, int device = 0, int precision = SC_PREC_FP32) {
    check(sc_plan_create_graph(m.nodes(), m.n_nodes(), m.edges(), m.n_edges(), m.weights(), m.n_weights(),
                               m.in_channels(), precision, device, &p_));
  }
  ~Plan() { sc_plan_destroy(p_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  int64_t ratio() const { int64_t r = 0; check(sc_plan_ratio(p_, &r)); return r; }
  int64_t latency() const { int64_t r = 0; check(sc_plan_latency(p_, &r)); return r; }
  int64_t state_bytes() const { int64_t r = 0; check(sc_plan_state_bytes(p_, &r)); return r; }
  void sink(int64_t* num, int64_t* den, int32_t* channels) const { check(sc_plan_sink_rate(p_, num, den, channels)); }
  const sc_plan* get() const { return p_; }

 private:
  sc_plan* p_ = nullptr;
};

class StreamBatch {  // StreamState for n independent streams
 public:
  StreamBatch(const Plan& plan, int n_streams, int64_t max_frames) {
    check(sc_state_create(plan.get(), n_streams, max_frames, &s_));
  }
  ~StreamBatch() { sc_state_destroy(s_); }
  StreamBatch(const StreamBatch&) = delete;
  StreamBatch& operator=(const StreamBatch&) = delete;

  // process_buffer for every stream; device pointers, async on `stream`
  void process_buffer(const float* d_in, float* d_out, int64_t frames, void* stream = nullptr) {
    check(sc_process(s_, d_in, d_out, frames, stream));
  }
  void reset(void* stream = nullptr) { check(sc_state_reset(s_, nullptr, 0, stream)); }
  void reset(const std::vector<int32_t>& ids, void* stream = nullptr) {
    check(sc_state_reset(s_, ids.data(), static_cast<int32_t>(ids.size()), stream));
  }

 private:
  sc_state* s_ = nullptr;
};

// ---- SPEC baseline_ola: overlap-add over the non-causal graph ---------
class OverlapAdd {
 public:
  OverlapAdd(const Graph& g, int64_t chunk, int overlap_pct, int n_streams, int64_t max_frames, int device = 0,
             int precision = SC_PREC_FP32) {
    Graph::Arrays a(g);
    check(sc_ola_create(a.n.data(), a.nn(), a.e.data(), a.ne(), g.weights().data(),
                        static_cast<int64_t>(g.weights().size()), g.in_channels(), precision, device, chunk,
                        overlap_pct, n_streams, max_frames, &o_));
  }
  ~OverlapAdd() { sc_ola_destroy(o_); }
  OverlapAdd(const OverlapAdd&) = delete;
  OverlapAdd& operator=(const OverlapAdd&) = delete;
  void process(const float* d_in, float* d_out, int64_t frames, void* stream = nullptr) {
    check(sc_ola_process(o_, d_in, d_out, frames, stream));
  }

 private:
  sc_ola* o_ = nullptr;
};

}  // namespace b200
}  // namespace streamconv
