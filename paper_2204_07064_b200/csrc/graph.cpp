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
  int64_t dly = 0;    // pending Delay: readers take rows shifted back by dly frames (DAG path)
  int zup = 1;        // pending ZeroUpsample factor: the next conv is a polyphase ConvT (DAG)
  int64_t dly_up = 0; // pending Delay after the ZeroUpsample, at the upsampled rate (DAG)
};

struct Lowerer {
  const sc_node* nodes;
  int n;
  const float* W;
  int64_t nW;
  Program* p;
  int pos = 0;
  int64_t ratio = 1;
  bool offline = false;  // original pads, no causalize delays (OLA per-chunk offline_run)

  static int64_t lcm(int64_t a, int64_t b) { return a / Rate::gcd(a, b) * b; }

  void need_cache(int buf, int64_t frames) {
    BufferSpec& b = p->bufs[buf];
    b.cache = std::max(b.cache, frames);
  }

  void need_tail(int buf, int64_t frames) {
    BufferSpec& b = p->bufs[buf];
    b.tail = std::max(b.tail, frames);
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

  // `shift`: right pad already folded into the left pad by causalize (ledger R = R + shift).
  void conv_node(const sc_node& nd, Value& v, int64_t shift = 0) {
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
    const int64_t L = nd.pad_left, R = nd.pad_right + shift, Ptot = L + nd.pad_right;
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
      op.look = emax + v.dly;  // a pending Delay (low rate) shifts the window back
      op.taps = static_cast<int>(emax + 1);
      op.row_step = 1;
      op.tap_step = 1;
      op.nout = static_cast<int>(r * N);
      op.w.assign(static_cast<size_t>(op.taps) * M * op.nout, 0.0f);
      op.bias.resize(op.nout);
      if (offline) {
        // original pad L on the zero-stuffed signal: y[r i + phi] = b + sum_k w[k] up[r i + phi
        // - L + k] with up[r m] = x[m]: phase phi takes the taps k = r e - phi + L at input row
        // i + e, e in [e_lo, e_hi] over all phases (e_hi > 0 reads rows past the chunk: zeros)
        int64_t elo = INT64_MAX, ehi = INT64_MIN;
        for (int phi = 0; phi < r; ++phi)
          for (int64_t k = 0; k < K; ++k) {
            const int64_t m = phi - L + k;
            if (((m % r) + r) % r) continue;
            const int64_t e = (m >= 0) ? m / r : -((-m) / r);
            elo = std::min(elo, e);
            ehi = std::max(ehi, e);
          }
        op.look = -elo + v.dly;
        op.taps = static_cast<int>(ehi - elo + 1);
        op.w.assign(static_cast<size_t>(op.taps) * M * op.nout, 0.0f);
        for (int phi = 0; phi < r; ++phi) {
          for (int q = 0; q < op.taps; ++q) {
            const int64_t k = r * (elo + q) - phi + L;
            if (k < 0 || k >= K) continue;
            for (int64_t c = 0; c < M; ++c)
              for (int64_t nn = 0; nn < N; ++nn)
                op.w[(static_cast<size_t>(q) * M + c) * op.nout + phi * N + nn] = w[(nn * M + c) * K + k];
          }
          for (int64_t nn = 0; nn < N; ++nn) op.bias[phi * N + nn] = b[nn];
        }
        need_tail(v.buf, std::max<int64_t>(0, ehi - v.dly));
      }
      for (int phi = 0; phi < r && !offline; ++phi) {
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
      need_cache(v.buf, op.look);
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
        Da = offline ? 0 : delay_for_stride(S, R, v.D);
        if (!offline && (v.D + R + Da) % S != 0) fail(SC_ERR_INTERNAL_NON_INTEGER_DELAY, "ledger division");
        v.D = offline ? 0 : (v.D + R + Da) / S;  // (offline programs keep no ledger)
        out_rate.den *= S;
        out_rate.norm();
        p->state_bytes_spec += M * Da * 4;  // inserted Delay(D_a) ring
      }
      p->state_bytes_spec += M * Ptot * 4;
      // A stride-S conv reads its input as S-frame super-rows (the polyphase view); its
      // window start must sit on a super-row boundary, so the look-back is rounded up to a
      // multiple of S and the kernel is front-padded with zero taps by the same shift.
      // a pending Delay (DAG path) widens the window look-back like an Eq. (2) delay does
      // offline: the original left pad only; rows past the chunk read as zeros (tail)
      const int64_t P = (offline ? L : Ptot + Da) + v.dly;
      if (offline) need_tail(v.buf, std::max<int64_t>(0, span - S - P));
      // (a dilated strided conv never runs on super-rows — the SIMT path reads it frame by
      // frame — and a zero-tap front pad would land on the wrong rows for d > 1)
      const int64_t Pa = (S > 1 && nd.dilation == 1) ? (P + S - 1) / S * S : P;
      const int64_t zshift = Pa - P;
      op.S = S;
      op.d = nd.dilation;
      op.look = Pa;
      op.taps = static_cast<int>(K + zshift);
      op.row_step = S;
      op.tap_step = nd.dilation;
      op.nout = nd.out_channels;
      op.w.assign(static_cast<size_t>(op.taps) * M * N, 0.0f);
      for (int64_t k = 0; k < K; ++k)
        for (int64_t c = 0; c < M; ++c)
          for (int64_t nn = 0; nn < N; ++nn)
            op.w[((k + zshift) * M + c) * N + nn] = w[(nn * M + c) * K + k];
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
    v.dly = 0;
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
          if (op.convt)  // r frames per polyphase row: use sc_plan_create_graph (SIMT sum)
            fail(SC_ERR_UNSUPPORTED_FORMAT, "a residual branch ending in a ConvTranspose1d (use the DAG API)");
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

// ================================================================== SPEC graph_ir (DAG)
// Exact rational for receptive-field extents (input samples).
struct Frac {
  int64_t n = 0, d = 1;
  Frac() = default;
  Frac(int64_t a, int64_t b = 1) : n(a), d(b) { norm(); }
  void norm() {
    if (d < 0) n = -n, d = -d;
    const int64_t g = Rate::gcd(n < 0 ? -n : n, d);
    if (g > 1) n /= g, d /= g;
  }
  Frac operator+(const Frac& o) const { return Frac(n * o.d + o.n * d, d * o.d); }
  Frac operator-(const Frac& o) const { return Frac(n * o.d - o.n * d, d * o.d); }
  bool operator<(const Frac& o) const { return n * o.d < o.n * d; }
  int64_t ceil() const { return n >= 0 ? (n + d - 1) / d : -((-n) / d); }
};

const char* gkind_name(int k) {
  static const char* names[] = {"Source", "Sink", "Conv", "ZeroUpsample", "Activation",
                                "Delay", "Sum", "Fanout", "Gate", "Slice"};
  return (k >= 0 && k <= SC_G_SLICE) ? names[k] : "?";
}

int g_inputs(const sc_gnode& g) {
  return g.kind == SC_G_SOURCE ? 0 : g.kind == SC_G_SUM ? g.arity : 1;
}
int g_outputs(const sc_gnode& g) {
  return g.kind == SC_G_SINK ? 0 : g.kind == SC_G_FANOUT ? g.arity : 1;
}

std::string nid(int i) { return "node " + std::to_string(i); }

}  // namespace

// validate: structure, acyclicity, reachability, channels, RateMap.
DagInfo dag_validate(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, int in_C) {
  if (n < 2 || !nodes) fail(SC_ERR_MALFORMED_GRAPH, "a graph needs a Source and a Sink");
  if (ne < 0 || (ne > 0 && !edges)) fail(SC_ERR_INVALID_ARGUMENT, "edge list");
  DagInfo g;
  for (int i = 0; i < n; ++i) {
    const sc_gnode& nd = nodes[i];
    switch (nd.kind) {
      case SC_G_SOURCE:
        if (g.source >= 0) fail(SC_ERR_MALFORMED_GRAPH, nid(i) + ": second Source (first is " + nid(g.source) + ")");
        g.source = i;
        break;
      case SC_G_SINK:
        if (g.sink >= 0) fail(SC_ERR_MALFORMED_GRAPH, nid(i) + ": second Sink (first is " + nid(g.sink) + ")");
        g.sink = i;
        break;
      case SC_G_CONV:
        if (nd.in_channels < 1 || nd.out_channels < 1 || nd.taps < 1 || nd.stride < 1 || nd.dilation < 1 ||
            nd.pad_left < 0 || nd.pad_right < 0 || nd.shift < 0)
          fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": Conv needs channels, kernel, stride, dilation >= 1 and pads >= 0");
        break;
      case SC_G_ZERO_UPSAMPLE:
        if (nd.factor < 1) fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": ZeroUpsample factor must be >= 1");
        break;
      case SC_G_ACTIVATION:
        if (nd.act < 0 || nd.act > 2) fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": unknown activation kind");
        break;
      case SC_G_DELAY:
        if (nd.samples < 0) fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": Delay samples must be >= 0");
        break;
      case SC_G_SUM:
      case SC_G_FANOUT:
        if (nd.arity < 2) fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": " + gkind_name(nd.kind) + " arity must be >= 2");
        break;
      case SC_G_GATE:
        break;
      case SC_G_SLICE:
        if (nd.slice_begin < 0 || nd.slice_count < 1) fail(SC_ERR_INVALID_ARGUMENT, nid(i) + ": slice range");
        break;
      default:
        fail(SC_ERR_SCHEMA_ERROR, nid(i) + ": unknown node kind " + std::to_string(nd.kind));
    }
  }
  if (g.source < 0) fail(SC_ERR_MALFORMED_GRAPH, "no Source node");
  if (g.sink < 0) fail(SC_ERR_MALFORMED_GRAPH, "no Sink node");
  g.in_edge.resize(n);
  g.out_edges.resize(n);
  for (int i = 0; i < n; ++i) g.in_edge[i].assign(g_inputs(nodes[i]), -1);
  for (int e = 0; e < ne; ++e) {
    const sc_edge& ed = edges[e];
    if (ed.from < 0 || ed.from >= n || ed.to < 0 || ed.to >= n)
      fail(SC_ERR_MALFORMED_GRAPH, "edge " + std::to_string(e) + " names a node outside 0.." + std::to_string(n - 1));
    if (ed.port < 0 || ed.port >= g_inputs(nodes[ed.to]))
      fail(SC_ERR_MALFORMED_GRAPH, "edge " + std::to_string(e) + ": " + nid(ed.to) + " (" + gkind_name(nodes[ed.to].kind) +
                                       ") has no input port " + std::to_string(ed.port));
    if (g.in_edge[ed.to][ed.port] >= 0)
      fail(SC_ERR_MALFORMED_GRAPH, nid(ed.to) + ": input port " + std::to_string(ed.port) + " has two edges");
    g.in_edge[ed.to][ed.port] = e;
    g.out_edges[ed.from].push_back(e);
  }
  for (int i = 0; i < n; ++i) {
    for (size_t q = 0; q < g.in_edge[i].size(); ++q)
      if (g.in_edge[i][q] < 0) fail(SC_ERR_DANGLING_NODE, nid(i) + ": input port " + std::to_string(q) + " is not connected");
    const int no = static_cast<int>(g.out_edges[i].size());
    if (no > g_outputs(nodes[i]))
      fail(SC_ERR_MALFORMED_GRAPH, nid(i) + " (" + gkind_name(nodes[i].kind) + ") has " + std::to_string(no) +
                                       " output edges (branching needs a Fanout of that arity)");
    if (no < g_outputs(nodes[i])) fail(SC_ERR_DANGLING_NODE, nid(i) + " (" + gkind_name(nodes[i].kind) + ") has an unconnected output");
  }
  // Kahn's algorithm: nodes left over sit on (or behind) a cycle
  std::vector<int> indeg(n);
  for (int i = 0; i < n; ++i) indeg[i] = static_cast<int>(g.in_edge[i].size());
  std::vector<int> ready;
  for (int i = n - 1; i >= 0; --i)
    if (indeg[i] == 0) ready.push_back(i);
  while (!ready.empty()) {
    const int u = ready.back();
    ready.pop_back();
    g.order.push_back(u);
    for (int e : g.out_edges[u])
      if (--indeg[edges[e].to] == 0) ready.push_back(edges[e].to);
  }
  if (static_cast<int>(g.order.size()) != n) {
    // report a node on the cycle: walk predecessors among the unordered nodes
    std::vector<char> done(n, 0);
    for (int u : g.order) done[u] = 1;
    int u = 0;
    while (done[u]) ++u;
    std::vector<int> seen(n, 0);
    while (!seen[u]) {
      seen[u] = 1;
      for (int e : g.in_edge[u])
        if (!done[edges[e].from]) { u = edges[e].from; break; }
    }
    fail(SC_ERR_CYCLE_DETECTED, nid(u) + " (" + gkind_name(nodes[u].kind) + ") lies on a cycle");
  }
  std::vector<char> fwd(n, 0), bwd(n, 0);
  fwd[g.source] = 1;
  for (int u : g.order)
    if (fwd[u])
      for (int e : g.out_edges[u]) fwd[edges[e].to] = 1;
  bwd[g.sink] = 1;
  for (int k = n - 1; k >= 0; --k) {
    const int u = g.order[k];
    for (int e : g.out_edges[u])
      if (bwd[edges[e].to]) bwd[u] = 1;
  }
  for (int i = 0; i < n; ++i) {
    if (!fwd[i]) fail(SC_ERR_DANGLING_NODE, nid(i) + " (" + gkind_name(nodes[i].kind) + ") is not reachable from the Source");
    if (!bwd[i]) fail(SC_ERR_DANGLING_NODE, "the Sink is not reachable from " + nid(i) + " (" + gkind_name(nodes[i].kind) + ")");
  }
  // channels and the RateMap along the topological order
  g.edge_C.assign(ne, 0);
  g.edge_rate.assign(ne, Rate{});
  for (int u : g.order) {
    const sc_gnode& nd = nodes[u];
    int C = 0;
    Rate r;
    if (nd.kind == SC_G_SOURCE) {
      C = nd.out_channels > 0 ? nd.out_channels : in_C;
      if (C < 1) fail(SC_ERR_INVALID_ARGUMENT, "Source channels must be >= 1");
      if (in_C > 0 && C != in_C)
        fail(SC_ERR_CHANNEL_MISMATCH, nid(u) + ": Source has " + std::to_string(C) + " channels, the call passes " + std::to_string(in_C));
    } else {
      const int e0 = g.in_edge[u][0];
      C = g.edge_C[e0];
      r = g.edge_rate[e0];
    }
    switch (nd.kind) {
      case SC_G_CONV:
        if (nd.in_channels != C)
          fail(SC_ERR_CHANNEL_MISMATCH, nid(u) + " (Conv) expects " + std::to_string(nd.in_channels) + " channels, gets " + std::to_string(C));
        C = nd.out_channels;
        r.den *= nd.stride;
        r.norm();
        break;
      case SC_G_ZERO_UPSAMPLE:
        r.num *= nd.factor;
        r.norm();
        break;
      case SC_G_SUM:
        for (int q = 1; q < nd.arity; ++q) {
          const int e = g.in_edge[u][q];
          if (g.edge_C[e] != C)
            fail(SC_ERR_CHANNEL_MISMATCH, nid(u) + " (Sum): input " + std::to_string(q) + " has " + std::to_string(g.edge_C[e]) +
                                              " channels, input 0 has " + std::to_string(C));
          if (g.edge_rate[e] != r)
            fail(SC_ERR_RATE_MISMATCH_AT_SUM, nid(u) + " (Sum): input " + std::to_string(q) + " runs at rate " +
                                                  std::to_string(g.edge_rate[e].num) + "/" + std::to_string(g.edge_rate[e].den) +
                                                  ", input 0 at " + std::to_string(r.num) + "/" + std::to_string(r.den));
        }
        break;
      case SC_G_GATE:
        if (C % 2) fail(SC_ERR_CHANNEL_MISMATCH, nid(u) + " (Gate) needs an even channel count");
        C /= 2;
        break;
      case SC_G_SLICE:
        if (nd.slice_begin + nd.slice_count > C) fail(SC_ERR_CHANNEL_MISMATCH, nid(u) + " (Slice) out of range");
        C = nd.slice_count;
        break;
      case SC_G_SINK:
        g.out_C = C;
        break;
      default:
        break;
    }
    for (int e : g.out_edges[u]) {
      g.edge_C[e] = C;
      g.edge_rate[e] = r;
      g.ratio = Lowerer::lcm(g.ratio, r.den);
    }
  }
  return g;
}

// receptive_field by interval propagation, exact rationals in input samples.
void dag_receptive_field(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, int in_C,
                         int64_t* past, int64_t* future) {
  const DagInfo g = dag_validate(nodes, n, edges, ne, in_C);
  std::vector<Frac> P(ne), F(ne);
  Frac po, fo;
  for (int u : g.order) {
    const sc_gnode& nd = nodes[u];
    Frac p, f;
    if (nd.kind != SC_G_SOURCE) {
      const int e0 = g.in_edge[u][0];
      p = P[e0];
      f = F[e0];
      const Rate r = g.edge_rate[e0];
      const Frac unit(r.den, r.num);  // input samples per frame of the incoming edge
      auto scale = [&](int64_t k) { return Frac(k * unit.n, unit.d); };
      if (nd.kind == SC_G_CONV) {
        // output frame i of a stride-S conv stands at the LAST input frame it consumes,
        // iS + S - 1 (streaming emits it once that frame has arrived); it reads input frames
        // [iS - L, iS - L + span - 1]
        const int64_t span = static_cast<int64_t>(nd.taps - 1) * nd.dilation + 1;
        p = p + scale(nd.pad_left + nd.stride - 1);
        f = f + scale(span - 1 - nd.pad_left - (nd.stride - 1));
      } else if (nd.kind == SC_G_DELAY) {
        p = p + scale(nd.samples);
        f = f - scale(nd.samples);
      } else if (nd.kind == SC_G_SUM) {
        for (int q = 1; q < nd.arity; ++q) {
          const int e = g.in_edge[u][q];
          if (p < P[e]) p = P[e];
          if (f < F[e]) f = F[e];
        }
      }
    }
    if (nd.kind == SC_G_SINK) po = p, fo = f;
    for (int e : g.out_edges[u]) P[e] = p, F[e] = f;
  }
  *past = std::max<int64_t>(0, po.ceil());
  *future = std::max<int64_t>(0, fo.ceil());
}

namespace {
// The causalize ledger over a validated DAG: D_c per edge at the edge's native
// rate, plus the delays causalize inserts (per edge: D_a before a strided conv, A_i at a Sum).
struct Ledger {
  std::vector<int64_t> D;       // cumulated delay per edge (before any inserted delay)
  std::vector<int64_t> insert;  // delay inserted on the edge
  int64_t sink_D = 0;
  int64_t latency_in = 0;
};

Ledger run_ledger(const sc_gnode* nodes, const sc_edge* edges, int ne, const DagInfo& g) {
  (void)edges;
  Ledger L;
  L.D.assign(ne, 0);
  L.insert.assign(ne, 0);
  for (int u : g.order) {
    const sc_gnode& nd = nodes[u];
    int64_t D = 0;
    if (nd.kind != SC_G_SOURCE) {
      const int e0 = g.in_edge[u][0];
      D = L.D[e0];
      switch (nd.kind) {
        case SC_G_CONV: {
          const int64_t R = nd.pad_right + nd.shift;
          if (nd.stride > 1) {
            const int64_t Da = delay_for_stride(nd.stride, R, D);  // Eq. (2)
            L.insert[e0] = Da;
            if ((D + R + Da) % nd.stride != 0) fail(SC_ERR_INTERNAL_NON_INTEGER_DELAY, nid(u) + ": ledger division");
            D = (D + R + Da) / nd.stride;
          } else {
            D += R;
          }
          break;
        }
        case SC_G_ZERO_UPSAMPLE:
          D *= nd.factor;
          break;
        case SC_G_DELAY:
          // only causalize-inserted Delays (D_a, A_i) enter the ledger: a Delay of the model
          // itself is part of its function in the original graph too, so it shifts both
          // graphs alike (counting it would misalign Sums and the latency)
          if (nd.inserted) D += nd.samples;
          break;
        case SC_G_SUM: {
          for (int q = 1; q < nd.arity; ++q) D = std::max(D, L.D[g.in_edge[u][q]]);
          for (int q = 0; q < nd.arity; ++q) {  // branch_alignment
            const int e = g.in_edge[u][q];
            L.insert[e] = D - L.D[e];
          }
          break;
        }
        default:
          break;
      }
    }
    if (nd.kind == SC_G_SINK) {
      L.sink_D = D;
      const Rate r = g.edge_rate[g.in_edge[u][0]];
      L.latency_in = D * r.den / r.num;
    }
    for (int e : g.out_edges[u]) L.D[e] = D;
  }
  return L;
}
}  // namespace

int64_t dag_causalize(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, int in_C,
                      std::vector<sc_gnode>* out_nodes, std::vector<sc_edge>* out_edges) {
  const DagInfo g = dag_validate(nodes, n, edges, ne, in_C);
  const Ledger L = run_ledger(nodes, edges, ne, g);
  if (out_nodes && out_edges) {
    out_nodes->assign(nodes, nodes + n);
    out_edges->clear();
    for (sc_gnode& nd : *out_nodes)
      if (nd.kind == SC_G_CONV) {  // pad (L, R) -> (L + R, 0)
        nd.shift += nd.pad_right;
        nd.pad_left += nd.pad_right;
        nd.pad_right = 0;
      }
    for (int e = 0; e < ne; ++e) {
      if (L.insert[e] == 0) {
        out_edges->push_back(edges[e]);
        continue;
      }
      sc_gnode dl{};
      dl.kind = SC_G_DELAY;
      dl.samples = L.insert[e];
      dl.inserted = 1;
      const int id = static_cast<int>(out_nodes->size());
      out_nodes->push_back(dl);
      out_edges->push_back(sc_edge{edges[e].from, id, 0});
      out_edges->push_back(sc_edge{id, edges[e].to, edges[e].port});
    }
  }
  return L.latency_in;
}

namespace {

// Lowering of a validated DAG onto the fused program: the Lowerer's conv lowering plus Delays
// as read offsets, ZeroUpsample + Conv as a polyphase ConvT, Sum as a residual epilogue or a
// SIMT sum launch, Fanout as shared readers (no fused epilogue on a fanned-out value).
struct DagLowerer {
  const sc_gnode* nodes;
  const sc_edge* edges;
  const DagInfo& g;
  Lowerer& lw;
  Program& p;
  std::vector<Value> val;  // per edge

  int writer_of(int buf) const {
    for (size_t i = 0; i < p.ops.size(); ++i)
      if (p.ops[i].out_buf == buf) return static_cast<int>(i);
    return -1;  // the source buffer (ingest)
  }

  void unsupported(int u, const std::string& why) {
    fail(SC_ERR_UNSUPPORTED_FORMAT, nid(u) + " (" + gkind_name(nodes[u].kind) + "): " + why);
  }

  void sum(int u, const sc_gnode& nd, Value& out) {
    std::vector<Value> in;
    int64_t Dmax = 0;
    for (int q = 0; q < nd.arity; ++q) {
      in.push_back(val[g.in_edge[u][q]]);
      if (in.back().zup > 1) unsupported(u, "a ZeroUpsample must feed a Conv");
      Dmax = std::max(Dmax, in.back().D);
    }
    std::vector<int64_t> eff(in.size());
    for (size_t q = 0; q < in.size(); ++q) {  // pending Delay + branch_alignment A_i
      const int64_t A = lw.offline ? 0 : Dmax - in[q].D;  // the original graph has no A_i
      eff[q] = in[q].dly + A;
      p.state_bytes_spec += static_cast<int64_t>(in[q].C) * A * 4;
    }
    if (nd.arity == 2) {
      // residual epilogue: the operand computed last is a conv output nobody else reads
      int j = -1, best = -1;
      for (int q = 0; q < 2; ++q) {
        const Value& v = in[q];
        if (v.producer < 0 || eff[q] != 0 || v.off != 0 || v.act != ACT_ID) continue;
        const ConvOp& op = p.ops[v.producer];
        // (a polyphase ConvT writes r frames per row: its epilogue has no per-frame residual)
        if (op.kind != OPK_CONV || op.convt || op.out_buf != v.buf || op.res_buf >= 0 || op.gate) continue;
        if (v.producer > best) best = v.producer, j = q;
      }
      if (j >= 0) {
        const Value& s = in[1 - j];
        if (writer_of(s.buf) < in[j].producer && s.buf != in[j].buf) {
          ConvOp& op = p.ops[in[j].producer];
          op.res_buf = s.buf;
          op.res_off = s.off;
          op.res_act = s.act;
          op.res_alpha = s.alpha;
          op.res_delay = eff[1 - j];
          lw.need_cache(s.buf, op.res_delay);
          out = in[j];
          out.D = Dmax;
          out.producer = -1;  // y = post(acc) + skip: a following act cannot fuse
          return;
        }
      }
    }
    if (nd.arity > 8) unsupported(u, "a Sum without a conv operand to absorb it takes at most 8 inputs");
    ConvOp op;
    op.kind = OPK_SUM;
    op.in_buf = in[0].buf;
    op.cin = in[0].C;
    op.nout = op.cout = op.out_rstride = in[0].C;
    op.in_rate = in[0].rate;
    for (size_t q = 0; q < in.size(); ++q) {
      SumIn si;
      si.buf = in[q].buf;
      si.off = in[q].off;
      si.act = in[q].act;
      si.alpha = in[q].alpha;
      si.delay = eff[q];
      lw.need_cache(si.buf, si.delay);
      op.sum_in.push_back(si);
    }
    op.name = "sum" + std::to_string(nd.arity) + " C" + std::to_string(in[0].C);
    op.out_buf = lw.new_buffer(in[0].C, in[0].rate, op.name);
    p.ops.push_back(std::move(op));
    out = in[0];
    out.buf = p.ops.back().out_buf;
    out.off = 0;
    out.act = ACT_ID;
    out.alpha = 0.f;
    out.dly = 0;
    out.D = Dmax;
    out.producer = static_cast<int>(p.ops.size()) - 1;
  }

  // Write the value (pending activation and Delay applied) to a buffer of its own with a
  // one-operand SIMT sum launch; `post` is applied on the store.
  void materialize(Value& v, int post, float post_alpha, const char* what) {
    ConvOp op;
    op.kind = OPK_SUM;
    op.in_buf = v.buf;
    op.cin = op.nout = op.cout = op.out_rstride = v.C;
    op.in_rate = v.rate;
    op.sum_in.push_back(SumIn{v.buf, v.off, v.act, v.alpha, v.dly});
    lw.need_cache(v.buf, v.dly);
    op.post_act = post;
    op.post_alpha = post_alpha;
    op.name = std::string(what) + " C" + std::to_string(v.C);
    op.out_buf = lw.new_buffer(v.C, v.rate, op.name);
    p.ops.push_back(std::move(op));
    v.buf = p.ops.back().out_buf;
    v.off = 0;
    v.act = ACT_ID;
    v.alpha = 0.f;
    v.dly = 0;
    v.producer = static_cast<int>(p.ops.size()) - 1;
  }

  void run() {
    for (int u : g.order) {
      const sc_gnode& nd = nodes[u];
      lw.pos = u + 1;  // error messages of the shared conv lowering name node ids
      Value v;
      if (nd.kind == SC_G_SOURCE) {
        v.C = p.in_C;
      } else if (nd.kind != SC_G_SUM) {
        v = val[g.in_edge[u][0]];
      }
      switch (nd.kind) {
        case SC_G_SOURCE:
        case SC_G_FANOUT:
          break;
        case SC_G_CONV: {
          // offline: a model Delay truncates its output at the chunk end, and a conv with right
          // padding must read zeros there, not the undelayed frames: materialise the delay
          if (lw.offline && v.dly > 0) materialize(v, ACT_ID, 0.f, "delay");
          sc_node c{};
          c.kind = SC_NODE_CONV;
          c.in_channels = nd.in_channels;
          c.out_channels = nd.out_channels;
          c.taps = nd.taps;
          c.stride = nd.stride;
          c.dilation = nd.dilation;
          c.pad_left = nd.pad_left;
          c.pad_right = nd.pad_right;
          c.weight_offset = nd.weight_offset;
          c.hint = nd.hint;
          if (v.zup > 1) {  // zero_upsample + conv = ConvTranspose1d
            if (nd.stride != 1 || nd.dilation != 1)
              unsupported(u, "a Conv after a ZeroUpsample must have stride 1 and dilation 1");
            if (v.dly_up % v.zup != 0)
              unsupported(u, "a Delay between ZeroUpsample and Conv must be a multiple of the factor");
            c.kind = SC_NODE_CONVT;
            c.stride = v.zup;
            const int64_t Dup = v.dly_up;
            v.dly += v.dly_up / v.zup;
            v.zup = 1;
            v.dly_up = 0;
            lw.conv_node(c, v, nd.shift);
            v.D += Dup;  // ledger: (D * s + Dup) + R
          } else {
            lw.conv_node(c, v, nd.shift);
          }
          break;
        }
        case SC_G_ZERO_UPSAMPLE:
          if (v.zup > 1) unsupported(u, "two ZeroUpsamples in a row");
          if (nd.factor > 1) v.zup = nd.factor;
          break;
        case SC_G_ACTIVATION: {
          if (nd.act == ACT_ID) break;
          const int pr = v.producer;
          if (pr >= 0 && p.ops[pr].post_act == ACT_ID && !p.ops[pr].gate && p.ops[pr].res_buf < 0 &&
              p.ops[pr].out_buf == v.buf && v.off == 0) {
            p.ops[pr].post_act = nd.act;  // fused epilogue activation
            p.ops[pr].post_alpha = nd.alpha;
          } else if (v.act == ACT_ID) {
            v.act = nd.act;  // applied by the consumer on load
            v.alpha = nd.alpha;
          } else {
            // a second activation on a value that already carries one: materialise
            // act2(act1(x)) with a one-operand SIMT sum launch (load act, store act)
            materialize(v, nd.act, nd.alpha, "act");
          }
          break;
        }
        case SC_G_DELAY:
          if (lw.offline && nd.inserted) break;  // absent from the original graph
          if (v.zup > 1) {
            v.dly_up += nd.samples;
          } else {
            v.dly += nd.samples;
            if (nd.inserted) v.D += nd.samples;  // ledger: causalize-inserted delays only
            p.state_bytes_spec += static_cast<int64_t>(v.C) * nd.samples * 4;  // Delay ring
          }
          break;
        case SC_G_SUM:
          sum(u, nd, v);
          break;
        case SC_G_GATE: {
          if (v.zup > 1 || v.dly != 0 || v.producer < 0 || p.ops[v.producer].kind != OPK_CONV ||
              p.ops[v.producer].post_act != ACT_ID || p.ops[v.producer].res_buf >= 0 || p.ops[v.producer].gate ||
              v.off != 0 || p.ops[v.producer].convt || p.ops[v.producer].out_buf != v.buf)
            unsupported(u, "a Gate must directly follow a stride-1 conv read by nothing else");
          ConvOp& op = p.ops[v.producer];
          const int H = op.nout / 2;
          std::vector<float> w2(op.w.size()), b2(op.nout);
          const size_t rows = op.w.size() / op.nout;
          for (size_t rr = 0; rr < rows; ++rr)
            for (int j = 0; j < H; ++j) {
              w2[rr * op.nout + 2 * j] = op.w[rr * op.nout + j];
              w2[rr * op.nout + 2 * j + 1] = op.w[rr * op.nout + H + j];
            }
          for (int j = 0; j < H; ++j) b2[2 * j] = op.bias[j], b2[2 * j + 1] = op.bias[H + j];
          op.w.swap(w2);
          op.bias.swap(b2);
          op.gate = true;
          op.out_rstride = H;
          p.bufs[op.out_buf].C = H;
          v.C = H;
          break;
        }
        case SC_G_SLICE:
          if (v.zup > 1) unsupported(u, "a ZeroUpsample must feed a Conv");
          v.off += nd.slice_begin;
          v.C = nd.slice_count;
          break;
        case SC_G_SINK:
          if (v.zup > 1) unsupported(u, "a ZeroUpsample must feed a Conv");
          p.sink_buf = v.buf;
          p.sink_off = v.off;
          p.sink_C = v.C;
          p.sink_act = v.act;
          p.sink_alpha = v.alpha;
          p.sink_rate = v.rate;
          p.sink_delay = v.dly;
          lw.need_cache(v.buf, v.dly);
          p.latency_sink = v.D;
          p.latency_in = v.D * v.rate.den / v.rate.num;
          break;
        default:
          break;
      }
      const int no = static_cast<int>(g.out_edges[u].size());
      for (int e : g.out_edges[u]) {
        val[e] = v;
        if (no > 1) val[e].producer = -1;  // a fanned-out value takes no fused epilogue
      }
    }
  }
};

}  // namespace

namespace {
bool densify4_disabled() {
  const char* e = std::getenv("SC_DENSIFY4");
  return e && std::atoi(e) == 0;  // SC_DENSIFY4=0: at most 2 output frames per row
}

bool densify_disabled() {
  const char* e = std::getenv("SC_DENSIFY");
  return e && std::atoi(e) == 0;  // SC_DENSIFY=0: keep narrow convs in their plain form
}

// Narrow stride-1 convs on the tensor cores waste most of a tile: N <= 64 columns (the MMA
// issue cost is per instruction, not per column) or a channel count padded to 32.  A
// densified op reads the input as 2-frame (4-frame for N <= 32) super-rows (the strided convs'
// view) and emits all output frames of a row at once, e.g. for two: y[2i + phi] = b + sum_k w[k] x[2i + phi - P + k] becomes one
// GEMM row with N' = 2N columns (phase-major) over the window's super-rows; MACs are unchanged
// for the padded-channel case and grow by (K + 1) / K otherwise.  Ops with a residual epilogue
// keep their form (their skip must stay in lockstep under phase state).
void densify(Program& p) {
  for (ConvOp& op : p.ops) {
    const BufferSpec& bi = p.bufs[op.in_buf];
    // stride S0 (1, or a strided conv already read as S0-frame super-rows): the densified op
    // reads 2 S0-frame super-rows and emits the two output frames 2i, 2i + 1 of each row
    const int S0 = op.S;
    if (op.kind != OPK_CONV || op.convt || op.tap_step != 1 || op.row_step != S0 || op.pqmf ||
        op.res_buf >= 0 || op.in_off != 0 || op.cin != bi.C || op.taps > 16 * S0 || op.nout > 1024 ||
        op.phases != 1 || op.d != 1)
      continue;
    const bool narrow = op.nout <= 64 || (S0 * op.cin % 32 != 0 && (2 * S0 * op.cin) % 32 == 0);
    // D output frames per row: 2, or 4 for the narrowest layers (N <= 32, e.g. the gated head:
    // N' = 4N fills a 128-column tile and a quarter fewer K-slabs cross the transform per frame)
    // when every non-phase call delivers a multiple of D S0 frames to this op
    auto even = [&](int D) {
      return (p.ratio * op.in_rate.num) % op.in_rate.den == 0 &&
             (p.ratio * op.in_rate.num / op.in_rate.den) % (D * S0) == 0;
    };
    if (!narrow || !even(2)) continue;
    const int D = (op.nout <= 32 && S0 == 1 && even(4) && !densify4_disabled()) ? 4 : 2;
    const int64_t extra = (D * S0 - op.look % (D * S0)) % (D * S0);  // window on a super-row boundary
    const int T0 = op.taps, N = op.nout, T1 = T0 + (D - 1) * S0 + static_cast<int>(extra);
    std::vector<float> w(static_cast<size_t>(T1) * op.cin * D * N, 0.f);
    for (int q = 0; q < T1; ++q)
      for (int ph = 0; ph < D; ++ph) {
        const int k = q - ph * S0 - static_cast<int>(extra);
        if (k < 0 || k >= T0) continue;
        for (int c = 0; c < op.cin; ++c)
          for (int n = 0; n < N; ++n)
            w[(static_cast<size_t>(q) * op.cin + c) * D * N + ph * N + n] =
                op.w[(static_cast<size_t>(k) * op.cin + c) * N + n];
      }
    op.w.swap(w);
    std::vector<float> b;
    for (int ph = 0; ph < D; ++ph) b.insert(b.end(), op.bias.begin(), op.bias.end());
    op.bias.swap(b);
    op.look += extra;
    op.taps = T1;
    op.S = D * S0;
    op.row_step = D * S0;
    op.phases = D;
    op.nout = D * N;
    op.out_rstride *= D;
    p.bufs[op.in_buf].cache = std::max(p.bufs[op.in_buf].cache, op.look);
    p.bufs[op.in_buf].align = Lowerer::lcm(p.bufs[op.in_buf].align, D * S0);
    op.name += D == 4 ? " x4" : " x2";
  }
}
}  // namespace

Program lower_dag(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
                  int64_t nW, int in_C, bool offline) {
  if (in_C < 1) fail(SC_ERR_INVALID_ARGUMENT, "in_channels must be >= 1");
  const DagInfo g = dag_validate(nodes, n, edges, ne, in_C);
  Program p;
  p.in_C = in_C;
  BufferSpec src;
  src.C = in_C;
  src.name = "source";
  p.bufs.push_back(src);
  sc_node dummy{};
  Lowerer lw{&dummy, 0, W, nW, &p};
  lw.offline = offline;
  p.offline = offline;
  DagLowerer dl{nodes, edges, g, lw, p, std::vector<Value>(ne)};
  dl.run();
  p.ratio = g.ratio;
  if (!offline && !densify_disabled()) densify(p);
  for (BufferSpec& b : p.bufs) b.cache = (b.cache + b.align - 1) / b.align * b.align;
  for (const ConvOp& op : p.ops) p.macs_per_sample += op.macs_per_sample;
  return p;
}

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
  p.ratio = lw.ratio;
  if (!densify_disabled()) densify(p);
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
  os << (offline ? "offline (original pads, per-call zero state)\n" : "") << "buffers:\n";
  for (size_t i = 0; i < bufs.size(); ++i)
    os << "  b" << i << " C=" << bufs[i].C << " cache=" << bufs[i].cache
       << (bufs[i].tail ? " tail=" + std::to_string(bufs[i].tail) : std::string()) << " rate=" << bufs[i].rate.num
       << "/" << bufs[i].rate.den << " (" << bufs[i].name << ")\n";
  os << "ops:\n";
  for (size_t i = 0; i < ops.size(); ++i) {
    const ConvOp& o = ops[i];
    if (o.kind == OPK_SUM) {
      os << "  op" << i << " " << o.name << " ->  b" << o.out_buf << " post=" << o.post_act << " =";
      for (const SumIn& si : o.sum_in)
        os << " b" << si.buf << "[" << si.off << ":+" << o.nout << "]@-" << si.delay << " act=" << si.act;
      os << "\n";
      continue;
    }
    os << "  op" << i << " " << o.name << " b" << o.in_buf << "[" << o.in_off << ":+" << o.cin
       << "] -> b" << o.out_buf << " look=" << o.look << " taps=" << o.taps << " nout=" << o.nout
       << " pre=" << o.pre_act << " post=" << o.post_act << (o.gate ? " gate" : "");
    if (o.res_buf >= 0) os << " +res(b" << o.res_buf << ", delay " << o.res_delay << ")";
    os << "\n";
  }
  os << "sink: b" << sink_buf << "[" << sink_off << ":+" << sink_C << "] act=" << sink_act
     << (sink_delay ? " delay=" + std::to_string(sink_delay) : std::string())
     << " rate=" << sink_rate.num << "/" << sink_rate.den << " ratio=" << ratio
     << " latency_sink=" << latency_sink << " state_bytes_spec=" << state_bytes_spec
     << " macs/sample=" << macs_per_sample << "\n";
  return os.str();
}

}  // namespace scb
