// graph.cpp — validate + causalize a node list and lower it to frame buffers and fused ops.
//
// Follows SPEC causalize: every Conv pad (L,R) becomes (L+R,0); before a
// stride-S conv an Eq. (2) delay D_a = (S - ((R + D_c) mod S)) mod S is inserted
// (SPEC.md:191-194); at a Sum the lower-delay branch gets A_i = max_j D_j - D_i
// (SPEC.md:200-204); the ledger maps conv D -> (D + R + D_a)/S, ZeroUpsample D -> D*s
// (SPEC.md:212).  Unlike the reference's node-per-op runtime, inserted
// Delays are not materialised: an Eq. (2) delay widens the conv's cache, and a skip Delay
// becomes a row offset into the residual input's own cache (no ring, no copy).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "program.hpp"

namespace scb {

namespace {

int64_t delay_for_stride(int64_t S, int64_t R, int64_t Dc) { return (S - ((R + Dc) % S)) % S; }

// ---- PQMF fast form (SC_HINT_PQMF): factor the cosine-modulated filter-bank weights.
// analysis (stride-M conv, 1 -> M, K taps): W[n][j], j = B*a + b (B = 2M): the modulation of
// band n repeats with period 2M in the tap index, so W[n][B a + b] = S[a][b] * Cm[n][b].
bool factor_pqmf_analysis(ConvOp& op, int M, int K) {
  const int B = 2 * M;
  if (K % B != 0 || op.cin != 1 || op.nout != M || op.taps != K) return false;
  const int A = K / B;
  auto W = [&](int n, int j) { return static_cast<double>(op.w[static_cast<size_t>(j) * M + n]); };
  double wmax = 0;
  for (float v : op.w) wmax = std::max(wmax, std::fabs(static_cast<double>(v)));
  std::vector<float> S(static_cast<size_t>(A) * B), Cm(static_cast<size_t>(M) * B);
  for (int b = 0; b < B; ++b) {
    int as = 0, ns = 0;
    double best = -1;
    for (int a = 0; a < A; ++a)
      for (int n = 0; n < M; ++n)
        if (std::fabs(W(n, B * a + b)) > best) best = std::fabs(W(n, B * a + b)), as = a, ns = n;
    if (best <= 0) return false;
    for (int n = 0; n < M; ++n) Cm[static_cast<size_t>(n) * B + b] = static_cast<float>(W(n, B * as + b) / W(ns, B * as + b));
    for (int a = 0; a < A; ++a) S[static_cast<size_t>(a) * B + b] = static_cast<float>(W(ns, B * a + b));
  }
  for (int n = 0; n < M; ++n)
    for (int a = 0; a < A; ++a)
      for (int b = 0; b < B; ++b) {
        const double rec = static_cast<double>(S[static_cast<size_t>(a) * B + b]) * Cm[static_cast<size_t>(n) * B + b];
        if (std::fabs(rec - W(n, B * a + b)) > 1e-6 * wmax) return false;
      }
  op.pqmf = 1;
  op.pq_A = A;
  op.pq_B = B;
  op.pq_M = M;
  op.pq_S.swap(S);
  op.pq_C.swap(Cm);
  return true;
}

// synthesis (polyphase ConvT M -> 1, r = M, Q taps over input frames): the weight vector over
// the M bands of every (q, phase) pair is proportional to one of <= 2M modulation vectors.
bool factor_pqmf_synthesis(ConvOp& op, int M) {
  const int Q = op.taps;
  if (op.cin != M || op.nout != M) return false;
  auto W = [&](int q, int c, int ph) { return static_cast<double>(op.w[(static_cast<size_t>(q) * M + c) * M + ph]); };
  double wmax = 0;
  for (float v : op.w) wmax = std::max(wmax, std::fabs(static_cast<double>(v)));
  std::vector<std::vector<double>> cls;  // normalized class vectors
  std::vector<int> idx(static_cast<size_t>(Q) * M, -1);
  std::vector<float> sval(static_cast<size_t>(Q) * M, 0.f);
  for (int q = 0; q < Q; ++q)
    for (int ph = 0; ph < M; ++ph) {
      int cm = 0;
      for (int c = 1; c < M; ++c)
        if (std::fabs(W(q, c, ph)) > std::fabs(W(q, cm, ph))) cm = c;
      const double piv = W(q, cm, ph);
      if (std::fabs(piv) <= 1e-30) continue;  // all-zero column: any class, s = 0 (idx stays -1)
      std::vector<double> v(M);
      for (int c = 0; c < M; ++c) v[c] = W(q, c, ph) / piv;
      int found = -1;
      for (size_t k = 0; k < cls.size() && found < 0; ++k) {
        // proportional up to sign: compare v with cls[k] scaled by its value at cm
        const double sc = cls[k][cm];
        if (std::fabs(sc) < 1e-3) continue;
        bool ok = true;
        for (int c = 0; c < M && ok; ++c) ok = std::fabs(cls[k][c] / sc - v[c]) <= 1e-5;
        if (ok) found = static_cast<int>(k);
      }
      if (found < 0) {
        cls.push_back(v);
        found = static_cast<int>(cls.size()) - 1;
        if (cls.size() > static_cast<size_t>(4 * M)) return false;
      }
      idx[static_cast<size_t>(q) * M + ph] = found;
      sval[static_cast<size_t>(q) * M + ph] = static_cast<float>(piv / cls[found][cm]);
    }
  if (cls.empty()) return false;
  // Canonical class order: with the cosine modulation the class of (q, phase) depends on q
  // only through q mod P (P = 2 for a 2M-periodic modulation) and, for a symmetric prototype,
  // on the phase only up to the mirror phase <-> M-1-phase.  Renumber the classes so that
  // class(q, phase) = (q mod P) * Mh + (mirror ? min(phase, M-1-phase) : phase), which lets
  // the kernel index them statically (and, mirrored, use each loaded class value twice).
  for (int cand = 0; cand < 6 && !op.pq_period; ++cand) {
    const int P = (cand % 3 == 0) ? 1 : (cand % 3 == 1) ? 2 : 4;
    const bool mirror = cand < 3;
    const int Mh = mirror ? M / 2 : M;
    if (Q % P != 0 || (mirror && M % 2) || cls.size() != static_cast<size_t>(P) * Mh) continue;
    auto slot_of = [&](int q, int ph) { return (q % P) * Mh + (mirror ? std::min(ph, M - 1 - ph) : ph); };
    std::vector<int> perm(cls.size(), -1), inv(cls.size(), -1);  // old class <-> canonical slot
    bool ok = true;
    for (int q = 0; q < Q && ok; ++q)
      for (int ph = 0; ph < M && ok; ++ph) {
        const int old = idx[static_cast<size_t>(q) * M + ph];
        if (old < 0) continue;
        const int slot = slot_of(q, ph);
        if (perm[old] < 0 && inv[slot] < 0) perm[old] = slot, inv[slot] = old;
        ok = perm[old] == slot && inv[slot] == old;
      }
    for (size_t k = 0; k < perm.size() && ok; ++k) ok = perm[k] >= 0;
    if (!ok) continue;
    std::vector<std::vector<double>> c2(cls.size());
    for (size_t k = 0; k < cls.size(); ++k) c2[perm[k]] = cls[k];
    cls.swap(c2);
    for (int q = 0; q < Q; ++q)
      for (int ph = 0; ph < M; ++ph) {
        int& v = idx[static_cast<size_t>(q) * M + ph];
        v = v < 0 ? slot_of(q, ph) : perm[v];
      }
    op.pq_period = P;
    op.pq_mirror = mirror ? 1 : 0;
  }
  for (int& v : idx) v = std::max(v, 0);
  std::vector<float> R(cls.size() * M);
  for (size_t k = 0; k < cls.size(); ++k)
    for (int c = 0; c < M; ++c) R[k * M + c] = static_cast<float>(cls[k][c]);
  for (int q = 0; q < Q; ++q)
    for (int ph = 0; ph < M; ++ph)
      for (int c = 0; c < M; ++c) {
        const size_t i = static_cast<size_t>(q) * M + ph;
        const double rec = static_cast<double>(sval[i]) * R[static_cast<size_t>(idx[i]) * M + c];
        if (std::fabs(rec - W(q, c, ph)) > 1e-6 * wmax) return false;
      }
  op.pqmf = 2;
  op.pq_A = Q;
  op.pq_B = static_cast<int>(cls.size());
  op.pq_M = M;
  op.pq_S.swap(sval);
  op.pq_C.swap(R);
  op.pq_idx.swap(idx);
  return true;
}

struct Value {
  int buf = 0;
  int off = 0;
  int C = 1;
  int act = ACT_ID;
  float alpha = 0.f;
  int producer = -1;  // op index that wrote it and may still take a fused epilogue
  Rate rate;
  int64_t D = 0;      // cumulated delay D_c, native rate
};

struct Lowerer {
  const sc_node* nodes;
  int n;
  const float* W;
  int64_t nW;
  Program* p;
  int pos = 0;
  int64_t ratio = 1;

  static int64_t lcm(int64_t a, int64_t b) { return a / Rate::gcd(a, b) * b; }

  void need_cache(int buf, int64_t frames) {
    BufferSpec& b = p->bufs[buf];
    b.cache = std::max(b.cache, frames);
  }

  void need_align(int buf, int64_t a) {
    BufferSpec& b = p->bufs[buf];
    b.align = lcm(b.align, a);
  }

  int new_buffer(int C, Rate rate, const std::string& name) {
    BufferSpec b;
    b.C = C;
    b.rate = rate;
    b.name = name;
    p->bufs.push_back(b);
    return static_cast<int>(p->bufs.size()) - 1;
  }

  void conv_node(const sc_node& nd, Value& v) {
    const bool convt = nd.kind == SC_NODE_CONVT;
    if (nd.in_channels < 1 || nd.out_channels < 1 || nd.taps < 1 || nd.stride < 1 ||
        nd.dilation < 1 || nd.pad_left < 0 || nd.pad_right < 0)
      fail(SC_ERR_INVALID_ARGUMENT, "conv node " + std::to_string(pos - 1) + ": bad shape");
    if (nd.in_channels != v.C)
      fail(SC_ERR_CHANNEL_MISMATCH, "conv node " + std::to_string(pos - 1) + " expects " +
                                        std::to_string(nd.in_channels) + " channels, got " +
                                        std::to_string(v.C));
    const int64_t M = nd.in_channels, N = nd.out_channels, K = nd.taps;
    const int64_t need = N * M * K + N;
    if (nd.weight_offset < 0 || nd.weight_offset + need > nW)
      fail(SC_ERR_INVALID_ARGUMENT, "conv node " + std::to_string(pos - 1) + ": weights out of range");
    const float* w = W + nd.weight_offset;
    const float* b = w + N * M * K;
    const int64_t L = nd.pad_left, R = nd.pad_right, Ptot = L + R;
    const int64_t span = (K - 1) * nd.dilation + 1;

    ConvOp op;
    op.convt = convt;
    op.in_buf = v.buf;
    op.in_off = v.off;
    op.cin = nd.in_channels;
    op.pre_act = v.act;
    op.pre_alpha = v.alpha;
    op.cout = nd.out_channels;
    op.K = nd.taps;
    op.in_rate = v.rate;
    Rate out_rate = v.rate;
    char nm[96];

    if (convt) {
      // ConvTranspose1d = zero_upsample(r) + conv1d(stride 1), lowered to
      // its polyphase form: y[r*i+phi] = b + sum_j w[k0(phi)+j*r] . x[i + j - e(phi)]
      const int r = nd.stride;
      if (nd.dilation != 1) fail(SC_ERR_INVALID_ARGUMENT, "convT dilation must be 1");
      if (Ptot != K - 1) fail(SC_ERR_PADDING_NOT_STREAMABLE, "convT pad must total K-1");
      const int64_t emax = (K - 1) / r;
      op.r = r;
      op.S = 1;
      op.d = 1;
      op.look = emax;
      op.taps = static_cast<int>(emax + 1);
      op.row_step = 1;
      op.tap_step = 1;
      op.nout = static_cast<int>(r * N);
      op.w.assign(static_cast<size_t>(op.taps) * M * op.nout, 0.0f);
      op.bias.resize(op.nout);
      for (int phi = 0; phi < r; ++phi) {
        const int64_t k0 = ((K - 1 - phi) % r + r) % r;
        const int64_t e = (K - 1 - phi - k0) / r;
        for (int q = 0; q < op.taps; ++q) {
          const int64_t k = k0 + (q + e - emax) * r;  // tap of the original kernel
          if (k < 0 || k >= K) continue;
          for (int64_t c = 0; c < M; ++c)
            for (int64_t nn = 0; nn < N; ++nn)
              op.w[(static_cast<size_t>(q) * M + c) * op.nout + phi * N + nn] =
                  w[(nn * M + c) * K + k];
        }
        for (int64_t nn = 0; nn < N; ++nn) op.bias[phi * N + nn] = b[nn];
      }
      need_cache(v.buf, emax);
      p->state_bytes_spec += M * Ptot * 4;   // SPEC: cache of the zero-stuffed signal
      v.D = v.D * r + R;                     // ledger: ZeroUpsample D*s, then conv + R
      out_rate.num *= r;
      out_rate.norm();
      // per input frame: r output frames x N x (K/r live taps) x M — no zero-stuffed MACs
      op.macs_per_sample = static_cast<double>(M) * N * K;
      std::snprintf(nm, sizeof nm, "convT%d %d->%d K%d", r, (int)M, (int)N, (int)K);
    } else {
      const int S = nd.stride;
      int64_t Da = 0;
      if (S == 1) {
        if (Ptot != span - 1)
          fail(SC_ERR_PADDING_NOT_STREAMABLE, "conv node " + std::to_string(pos - 1) +
                                                  ": pad must total (K-1)*d");
        v.D += R;
      } else {
        if (Ptot < span - S)
          fail(SC_ERR_PADDING_NOT_STREAMABLE, "strided conv: pad must be >= span - stride");
        Da = delay_for_stride(S, R, v.D);
        if ((v.D + R + Da) % S != 0) fail(SC_ERR_INTERNAL_NON_INTEGER_DELAY, "ledger division");
        v.D = (v.D + R + Da) / S;
        out_rate.den *= S;
        out_rate.norm();
        p->state_bytes_spec += M * Da * 4;  // inserted Delay(D_a) ring
      }
      p->state_bytes_spec += M * Ptot * 4;
      // A stride-S conv reads its input as S-frame super-rows (the polyphase view); its
      // window start must sit on a super-row boundary, so the look-back is rounded up to a
      // multiple of S and the kernel is front-padded with zero taps by the same shift.
      const int64_t P = Ptot + Da;
      const int64_t Pa = (S > 1) ? (P + S - 1) / S * S : P;
      const int64_t shift = Pa - P;
      op.S = S;
      op.d = nd.dilation;
      op.look = Pa;
      op.taps = static_cast<int>(K + shift);
      op.row_step = S;
      op.tap_step = nd.dilation;
      op.nout = nd.out_channels;
      op.w.assign(static_cast<size_t>(op.taps) * M * N, 0.0f);
      for (int64_t k = 0; k < K; ++k)
        for (int64_t c = 0; c < M; ++c)
          for (int64_t nn = 0; nn < N; ++nn)
            op.w[((k + shift) * M + c) * N + nn] = w[(nn * M + c) * K + k];
      op.bias.assign(b, b + N);
      need_cache(v.buf, op.look);
      if (S > 1) need_align(v.buf, S);
      op.macs_per_sample = static_cast<double>(M) * N * K / S;  // per input frame
      std::snprintf(nm, sizeof nm, "conv%s %d->%d K%d d%d", S > 1 ? ("/" + std::to_string(S)).c_str() : "",
                    (int)M, (int)N, (int)K, nd.dilation);
    }
    if (nd.hint == SC_HINT_PQMF) {
      if (convt && nd.out_channels == 1 && nd.stride == nd.in_channels) factor_pqmf_synthesis(op, nd.in_channels);
      if (!convt && nd.in_channels == 1 && nd.stride == nd.out_channels && op.look == Ptot)
        factor_pqmf_analysis(op, nd.out_channels, nd.taps);
      if (op.pqmf) std::snprintf(nm, sizeof nm, "pqmf-%s %d bands K%d", convt ? "synthesis" : "analysis",
                                 convt ? nd.in_channels : nd.out_channels, (int)K);
      if (op.pqmf == 2 && op.pq_period) std::snprintf(nm + std::strlen(nm), sizeof nm - std::strlen(nm), " P%d%s", op.pq_period,
                                              op.pq_mirror ? "m" : "");
    }
    op.name = nm;
    // scale per-input-frame MACs to per-input-SAMPLE of the model
    op.macs_per_sample *= static_cast<double>(v.rate.num) / static_cast<double>(v.rate.den);
    op.out_rstride = op.nout;
    ratio = lcm(ratio, out_rate.den);
    op.out_buf = new_buffer(nd.out_channels, out_rate, op.name);
    p->ops.push_back(std::move(op));
    v.buf = p->ops.back().out_buf;
    v.off = 0;
    v.C = nd.out_channels;
    v.act = ACT_ID;
    v.alpha = 0.f;
    v.producer = static_cast<int>(p->ops.size()) - 1;
    v.rate = out_rate;
  }

  void parse(Value& v, int depth) {
    while (pos < n) {
      const sc_node& nd = nodes[pos];
      if (nd.kind == SC_NODE_RES_END) {
        if (depth == 0) fail(SC_ERR_MALFORMED_GRAPH, "RES_END without RES_BEGIN at node " + std::to_string(pos));
        return;
      }
      ++pos;
      switch (nd.kind) {
        case SC_NODE_CONV:
        case SC_NODE_CONVT:
          conv_node(nd, v);
          break;
        case SC_NODE_ACT: {
          if (nd.act < 0 || nd.act > 2) fail(SC_ERR_INVALID_ARGUMENT, "activation kind");
          if (nd.act == ACT_ID) break;
          if (v.producer >= 0 && p->ops[v.producer].post_act == ACT_ID &&
              !p->ops[v.producer].gate && p->ops[v.producer].res_buf < 0 &&
              p->ops[v.producer].out_buf == v.buf) {
            // fused epilogue activation of the producing conv
            p->ops[v.producer].post_act = nd.act;
            p->ops[v.producer].post_alpha = nd.alpha;
          } else if (v.act == ACT_ID) {
            v.act = nd.act;  // pending: applied by the consumer on load (prologue)
            v.alpha = nd.alpha;
          } else {
            fail(SC_ERR_UNSUPPORTED_FORMAT, "two unfused activations in a row");
          }
          break;
        }
        case SC_NODE_GATE: {
          if (v.C % 2) fail(SC_ERR_CHANNEL_MISMATCH, "gate needs an even channel count");
          if (v.producer < 0 || p->ops[v.producer].post_act != ACT_ID ||
              p->ops[v.producer].res_buf >= 0 || p->ops[v.producer].gate || v.off != 0 ||
              p->ops[v.producer].convt)
            fail(SC_ERR_UNSUPPORTED_FORMAT, "gate must directly follow a stride-1 conv");
          ConvOp& op = p->ops[v.producer];
          // interleave columns: new col 2j = wave j, 2j+1 = amp j
          const int H = op.nout / 2;
          std::vector<float> w2(op.w.size()), b2(op.nout);
          const size_t rows = op.w.size() / op.nout;
          for (size_t rr = 0; rr < rows; ++rr)
            for (int j = 0; j < H; ++j) {
              w2[rr * op.nout + 2 * j] = op.w[rr * op.nout + j];
              w2[rr * op.nout + 2 * j + 1] = op.w[rr * op.nout + H + j];
            }
          for (int j = 0; j < H; ++j) {
            b2[2 * j] = op.bias[j];
            b2[2 * j + 1] = op.bias[H + j];
          }
          op.w.swap(w2);
          op.bias.swap(b2);
          op.gate = true;
          op.out_rstride = H;
          p->bufs[op.out_buf].C = H;
          v.C = H;
          break;
        }
        case SC_NODE_SLICE: {
          if (nd.slice_begin < 0 || nd.slice_count < 1 || nd.slice_begin + nd.slice_count > v.C)
            fail(SC_ERR_CHANNEL_MISMATCH, "slice out of range");
          v.off += nd.slice_begin;
          v.C = nd.slice_count;
          break;
        }
        case SC_NODE_RES_BEGIN: {
          Value skip = v;
          Value br = v;
          br.producer = -1;  // the branch input is shared with the skip: no fused epilogue
          parse(br, depth + 1);
          if (pos >= n || nodes[pos].kind != SC_NODE_RES_END)
            fail(SC_ERR_MALFORMED_GRAPH, "RES_BEGIN without RES_END");
          ++pos;
          if (br.C != skip.C) fail(SC_ERR_CHANNEL_MISMATCH, "residual branch changes channels");
          if (br.rate != skip.rate) fail(SC_ERR_RATE_MISMATCH_AT_SUM, "residual rates differ");
          const int64_t Dmax = std::max(br.D, skip.D);  // branch_alignment
          if (Dmax != br.D) fail(SC_ERR_UNSUPPORTED_FORMAT, "branch-side alignment delay");
          if (br.producer < 0 || br.act != ACT_ID || br.off != 0 || br.buf != p->ops[br.producer].out_buf)
            fail(SC_ERR_UNSUPPORTED_FORMAT, "residual branch must end with a conv");
          ConvOp& op = p->ops[br.producer];
          if (op.res_buf >= 0 || op.gate) fail(SC_ERR_UNSUPPORTED_FORMAT, "residual epilogue busy");
          op.res_buf = skip.buf;
          op.res_off = skip.off;
          op.res_act = skip.act;
          op.res_alpha = skip.alpha;
          op.res_delay = Dmax - skip.D;
          need_cache(skip.buf, op.res_delay);
          p->state_bytes_spec += static_cast<int64_t>(skip.C) * op.res_delay * 4;
          v = br;
          v.D = Dmax;
          v.producer = -1;  // y = post(acc) + skip: a following act cannot fuse
          break;
        }
        default:
          fail(SC_ERR_SCHEMA_ERROR, "unknown node kind " + std::to_string(nd.kind) + " at node " +
                                        std::to_string(pos - 1));
      }
    }
    if (depth > 0) fail(SC_ERR_MALFORMED_GRAPH, "RES_BEGIN without RES_END");
  }
};

}  // namespace

Program lower_graph(const sc_node* nodes, int n_nodes, const float* W, int64_t nW, int in_C) {
  if (in_C < 1) fail(SC_ERR_INVALID_ARGUMENT, "in_channels must be >= 1");
  if (n_nodes < 0 || (n_nodes > 0 && !nodes)) fail(SC_ERR_INVALID_ARGUMENT, "node list");
  Program p;
  p.in_C = in_C;
  BufferSpec src;
  src.C = in_C;
  src.name = "source";
  p.bufs.push_back(src);
  Lowerer lw{nodes, n_nodes, W, nW, &p};
  Value v;
  v.C = in_C;
  lw.parse(v, 0);
  for (BufferSpec& b : p.bufs) b.cache = (b.cache + b.align - 1) / b.align * b.align;
  p.sink_buf = v.buf;
  p.sink_off = v.off;
  p.sink_C = v.C;
  p.sink_act = v.act;
  p.sink_alpha = v.alpha;
  p.sink_rate = v.rate;
  p.ratio = lw.ratio;
  p.latency_sink = v.D;
  p.latency_in = v.D * v.rate.den / v.rate.num;
  for (const ConvOp& op : p.ops) p.macs_per_sample += op.macs_per_sample;
  return p;
}

std::string Program::describe() const {
  std::ostringstream os;
  os << "buffers:\n";
  for (size_t i = 0; i < bufs.size(); ++i)
    os << "  b" << i << " C=" << bufs[i].C << " cache=" << bufs[i].cache << " rate=" << bufs[i].rate.num
       << "/" << bufs[i].rate.den << " (" << bufs[i].name << ")\n";
  os << "ops:\n";
  for (size_t i = 0; i < ops.size(); ++i) {
    const ConvOp& o = ops[i];
    os << "  op" << i << " " << o.name << " b" << o.in_buf << "[" << o.in_off << ":+" << o.cin
       << "] -> b" << o.out_buf << " look=" << o.look << " taps=" << o.taps << " nout=" << o.nout
       << " pre=" << o.pre_act << " post=" << o.post_act << (o.gate ? " gate" : "");
    if (o.res_buf >= 0) os << " +res(b" << o.res_buf << ", delay " << o.res_delay << ")";
    os << "\n";
  }
  os << "sink: b" << sink_buf << "[" << sink_off << ":+" << sink_C << "] act=" << sink_act
     << " rate=" << sink_rate.num << "/" << sink_rate.den << " ratio=" << ratio
     << " latency_sink=" << latency_sink << " state_bytes_spec=" << state_bytes_spec
     << " macs/sample=" << macs_per_sample << "\n";
  return os.str();
}

}  // namespace scb
