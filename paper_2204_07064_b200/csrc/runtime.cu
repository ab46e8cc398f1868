// runtime.cu — plans, stream states and the per-call launch sequence (the stream_runtime).
//
// A plan is the causalized, lowered model with device-resident weights (one per device).  A
// state is SPEC's StreamState for a whole batch of independent streams:
// every activation buffer [stream][cache + T][C] lives in HBM; the first `cache` frames of
// each buffer ARE the cached padding.  One call (process_buffer) is:
//   ingest(x) -> fused cached-conv ops in topological order -> egress(y) -> carry(caches)
// replayed from a CUDA graph captured once per buffer length.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "program.hpp"
#include "runtime.hpp"

namespace scb {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(SC_ERR_CUDA_BASE + static_cast<int>(e), std::string(what) + ": " + cudaGetErrorString(e));
}
int64_t round_up(int64_t a, int64_t m) { return (a + m - 1) / m * m; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q), "GetDriverEntryPoint");
    if (q != cudaDriverEntryPointSuccess || !f) fail(SC_ERR_CUDA_BASE, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 3-D tensor map (fp32 with 128B swizzle: inner box = 32 floats = 128 bytes; or bf16 with
// 64B swizzle: inner box = 32 bf16 = 64 bytes).
CUtensorMap make_map3(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                      uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2, bool bf16 = false,
                      bool fp16 = false) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           (bf16 || fp16) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(SC_ERR_CUDA_BASE, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

bool pqmf_disabled() {
  const char* e = std::getenv("SC_DISABLE_PQMF");
  return e && std::atoi(e) != 0;
}

int graphs_per_plan() {
  static int n = 0;
  if (n == 0) {
    const char* e = std::getenv("SC_GRAPHS_PER_PLAN");
    n = std::max(1, e ? std::atoi(e) : 1);
  }
  return n;
}

// bf16 plans keep the residual stream (buffers read as a residual skip or written by a
// residual epilogue) in fp32 unless SC_BF16_SKIP=bf16: rounding the running sum to bf16 at
// every unit compounds over cfg4/cfg5's 12-27 residual units (nrmse 4.6e-2 at cfg4's literal
// init), while the conv operands are rounded by the transform warps anyway.
bool bf16_skip_fp32() {
  const char* e = std::getenv("SC_BF16_SKIP");
  return !(e && std::string(e) == "bf16");
}

bool bf16_store_disabled() {
  const char* e = std::getenv("SC_BF16_STORE");
  return e && std::atoi(e) == 0;  // SC_BF16_STORE=0: keep every buffer fp32 in bf16 plans
}

bool win_disabled() {
  const char* e = std::getenv("SC_DISABLE_WIN");
  return e && std::atoi(e) != 0;
}

// fp32 plans: the fp32-accurate tensor-core split — "f16" (3xFP16, default) or "tf32" (3xTF32,
// the round-1 form; chained k3 + 1x1 convs always use it).  SC_FP32_SPLIT=tf32 selects it.
bool split_tf32() {
  const char* e = std::getenv("SC_FP32_SPLIT");
  return e && std::string(e) == "tf32";
}

// 3xFP16 non-window tiles: per-block input windows (TcParams::awin); SC_AWIN=0 disables
bool awin_disabled() {
  const char* e = std::getenv("SC_AWIN");
  return e && e[0] == '0';
}

bool io_fuse_disabled() {  // SC_IO_FUSE=0: keep the ingest / egress launches
  const char* e = std::getenv("SC_IO_FUSE");
  return e && e[0] == '0';
}

bool small_bn_disabled() {
  const char* e = std::getenv("SC_SMALL_BN");
  return e && e[0] == '0';
}

bool tc_disabled() {
  const char* e = std::getenv("SC_DISABLE_TC");
  return e && std::atoi(e) != 0;
}

// Decide whether an op runs on the tensor-core kernel and build its hi/lo weight planes.
void plan_tc(const Program& pg, size_t i, int precision, DevOp& d, std::vector<float>& wtc, bool f16 = false) {
  const ConvOp& op = pg.ops[i];
  if (op.kind == OPK_SUM) {
    d.kernel = KERNEL_SUM;
    return;
  }
  const BufferSpec& bi = pg.bufs[op.in_buf];
  const bool strided = !op.convt && op.S > 1;
  const int S = strided ? op.S : 1;
  const int cin_view = S * op.cin;
  const int bufC_view = S * bi.C;
  bool ok = !tc_disabled() && op.nout % 32 == 0 && op.nout <= 2048 &&
            cin_view >= 16 &&
            bufC_view % 4 == 0;
  if (strided) ok = ok && op.in_off == 0 && op.cin == bi.C && op.d == 1;
  if (!ok) return;
  if (op.gate) {
    // the output tile (BN/2 columns) is stored as 32-column TMA boxes clipped at the buffer
    // width: a partial box is only allowed as the last (and only) one
    if (op.nout > 64 && op.nout % 64 != 0) return;
    d.BN = (op.nout % 128 == 0) ? 128 : (op.nout % 64 == 0) ? 64 : 32;
  } else {
    d.BN = (op.nout % 128 == 0) ? 128 : (op.nout % 64 == 0) ? 64 : 32;
  }
  if (op.out_rstride % 4 != 0 || (op.res_buf >= 0 && (pg.bufs[op.res_buf].C % 4 != 0 || op.res_off % 4 != 0)))
    return;
  d.kernel = KERNEL_TC;
  d.bf16 = precision == SC_PREC_BF16;
  d.view_S = S;
  d.cin_view = cin_view;
  d.cin_view_pad = static_cast<int>(round_up(cin_view, 32));
  d.taps_view = strided ? static_cast<int>((op.taps + S - 1) / S) : op.taps;
  d.tap_rows = strided ? 1 : op.tap_step;
  const int64_t Kpad = static_cast<int64_t>(d.taps_view) * d.cin_view_pad;
  const int64_t N = op.nout;
  d.f16 = f16 && !d.bf16;
  // 3xFP16: one power-of-two scale per layer puts max |w| in [2^14, 2^15) (kernels_tc.cu HF)
  d.f16_sw = 0;
  if (d.f16) {
    float wmax = 0.f;
    for (float w : op.w) wmax = std::max(wmax, std::fabs(w));
    const int e = wmax > 0.f ? std::ilogb(wmax) : 0;
    d.f16_sw = std::min(100, std::max(-100, 14 - e));
  }
  const float wsc = std::ldexp(1.0f, d.f16_sw);
  // fp32: [2 (hi, lo)][N][Kpad] floats; bf16: [N][Kpad] bf16 (round-to-nearest) packed in floats;
  // 3xFP16: [2 (hi, lo)][N][Kpad] fp16 of w x 2^f16_sw (packed two per float slot)
  wtc.assign(d.bf16 ? static_cast<size_t>((N * Kpad + 1) / 2) : d.f16 ? static_cast<size_t>(N * Kpad)
                                                                     : static_cast<size_t>(2 * N * Kpad), 0.f);
  uint16_t* wb = reinterpret_cast<uint16_t*>(wtc.data());
  for (int64_t n = 0; n < N; ++n)
    for (int q = 0; q < d.taps_view; ++q)
      for (int cv = 0; cv < cin_view; ++cv) {
        float w;
        if (strided) {
          const int rho = cv / op.cin, c = cv % op.cin;
          const int k = q * S + rho;
          w = (k < op.taps) ? op.w[(static_cast<size_t>(k) * op.cin + c) * N + n] : 0.f;
        } else {
          w = op.w[(static_cast<size_t>(q) * op.cin + cv) * N + n];
        }
        const size_t o = static_cast<size_t>(n) * Kpad + static_cast<size_t>(q) * d.cin_view_pad + cv;
        if (d.bf16) {
          const uint32_t u = __builtin_bit_cast(uint32_t, w);
          wb[o] = static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);  // RN-even
        } else if (d.f16) {
          const float ws = w * wsc;  // exact (power of two)
          const __half h = __float2half_rn(ws);
          const __half l = __float2half_rn(ws - __half2float(h));
          wb[o] = __half_as_ushort(h);
          wb[static_cast<size_t>(N * Kpad) + o] = __half_as_ushort(l);
        } else {
          const float hi = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, w) & 0xFFFFE000u);
          wtc[o] = hi;
          wtc[static_cast<size_t>(N * Kpad) + o] = w - hi;
        }
      }
}
}  // namespace

// the chained GEMM (K = 128) accumulates in one TMEM chunk (3% faster on cfg2: three fewer
// chunk drains per tile; max error 1.4e-5 x RMS vs 7.9e-6) unless SC_CHAIN_ONE=0, which keeps
// per-slab chunks — bit-identical to the two-launch form (tests/test_gpu_chain.py)
int chain_one() {
  const char* e = std::getenv("SC_CHAIN_ONE");
  return e && e[0] == '0' ? 0 : 1;
}

bool chain_disabled() {
  const char* e = std::getenv("SC_CHAIN");
  return e && e[0] == '0';
}

// Chained 1x1 convs (fp32 tensor-core path): a BN = 128 conv whose output buffer is read only
// by the next op, a K = 1 conv over the same 128 channels, runs both GEMMs in one launch — the
// intermediate tile never leaves the SM (kernels_tc.cu CH; cfg2's residual blocks: LReLU ->
// conv K3 -> LReLU -> conv 1x1 + skip).  The 1x1 weights are appended along K of the first
// conv's packed weights ([2][128][Kpad + 128]), so one weight map serves both GEMMs.
// merge = false: only mark the chain-eligible pairs (DevOp::chain) without touching weights —
// fp32 plans keep such pairs on the 3xTF32 split even when SC_CHAIN=0, so the two-launch form
// stays bit-identical to the chained one
void find_chains(const Program& pg, std::vector<DevOp>& dops, std::vector<std::vector<float>>& wtc,
                 bool merge = true) {
  for (size_t i = 0; i + 1 < pg.ops.size(); ++i) {
    const size_t j = i + 1;
    const ConvOp& a = pg.ops[i];
    const ConvOp& b = pg.ops[j];
    DevOp& da = dops[i];
    const DevOp& db = dops[j];
    if (da.kernel != KERNEL_TC || db.kernel != KERNEL_TC || da.bf16 != db.bf16 || da.chain >= 0) continue;
    if (da.BN != 128 || db.BN != 128 || da.view_S != 1 || db.view_S != 1 || db.taps_view != 1) continue;
    if (a.kind != OPK_CONV || b.kind != OPK_CONV || a.convt || b.convt || a.phases != 1 || b.phases != 1) continue;
    if (a.nout != 128 || a.out_rstride != 128 || pg.bufs[a.out_buf].C != 128 || a.gate || a.res_buf >= 0) continue;
    if (a.post_act == ACT_TANH || b.pre_act == ACT_TANH) continue;
    if (b.in_buf != a.out_buf || b.in_off != 0 || b.cin != 128 || b.look != 0 || b.nout != 128 || b.gate) continue;
    if (b.out_buf == a.out_buf || b.res_buf == a.out_buf || a.out_buf == pg.sink_buf) continue;
    bool other = false;  // the intermediate buffer has no other reader
    for (size_t k = 0; k < pg.ops.size() && !other; ++k) {
      if (k == j) continue;
      const ConvOp& o = pg.ops[k];
      other = o.in_buf == a.out_buf || o.res_buf == a.out_buf;
      for (const SumIn& si : o.sum_in) other = other || si.buf == a.out_buf;
    }
    if (other) continue;
    if (!merge) {
      da.chain = static_cast<int>(j);
      continue;
    }
    const size_t N = 128, K1 = static_cast<size_t>(da.taps_view) * da.cin_view_pad, K2 = 128;
    std::vector<float> w;
    if (da.bf16) {  // [N][K] bf16 (packed two per float slot)
      w.assign((N * (K1 + K2) + 1) / 2, 0.f);
      const uint16_t* w1 = reinterpret_cast<const uint16_t*>(wtc[i].data());
      const uint16_t* w2 = reinterpret_cast<const uint16_t*>(wtc[j].data());
      uint16_t* o = reinterpret_cast<uint16_t*>(w.data());
      for (size_t n = 0; n < N; ++n) {
        std::copy_n(w1 + n * K1, K1, o + n * (K1 + K2));
        std::copy_n(w2 + n * K2, K2, o + n * (K1 + K2) + K1);
      }
    } else {  // [2 (hi, lo)][N][K] fp32
      w.assign(2 * N * (K1 + K2), 0.f);
      for (size_t h = 0; h < 2; ++h)
        for (size_t n = 0; n < N; ++n) {
          std::copy_n(wtc[i].begin() + (h * N + n) * K1, K1, w.begin() + (h * N + n) * (K1 + K2));
          std::copy_n(wtc[j].begin() + (h * N + n) * K2, K2, w.begin() + (h * N + n) * (K1 + K2) + K1);
        }
    }
    wtc[i] = std::move(w);
    da.chain = static_cast<int>(j);
    da.k_chain = static_cast<int>(K2);
    da.chain_one = chain_one();
  }
}

Plan::~Plan() {
  if (wmem && device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(wmem);
    cudaSetDevice(prev);
  }
}

std::unique_ptr<Plan> make_plan(const sc_node* nodes, int n_nodes, const float* W, int64_t nW,
                                int in_C, int precision, int device) {
  if (precision != SC_PREC_FP32 && precision != SC_PREC_BF16)
    fail(SC_ERR_INVALID_ARGUMENT, "precision must be SC_PREC_FP32 or SC_PREC_BF16");
  if (n_nodes > 0 && !W && nW > 0) fail(SC_ERR_INVALID_ARGUMENT, "weights pointer is null");
  return make_plan(lower_graph(nodes, n_nodes, W, nW, in_C), precision, device);
}

std::unique_ptr<Plan> make_plan_dag(const sc_gnode* nodes, int n_nodes, const sc_edge* edges,
                                    int n_edges, const float* W, int64_t nW, int in_C,
                                    int precision, int device) {
  if (precision != SC_PREC_FP32 && precision != SC_PREC_BF16)
    fail(SC_ERR_INVALID_ARGUMENT, "precision must be SC_PREC_FP32 or SC_PREC_BF16");
  if (!W && nW > 0) fail(SC_ERR_INVALID_ARGUMENT, "weights pointer is null");
  return make_plan(lower_dag(nodes, n_nodes, edges, n_edges, W, nW, in_C), precision, device);
}

std::unique_ptr<Plan> make_plan(Program prog, int precision, int device) {
  auto plan = std::make_unique<Plan>();
  plan->prog = std::move(prog);
  plan->precision = precision;
  plan->device = device;
  plan->desc = plan->prog.describe();
  if (device == -1) return plan;  // host-only plan: lowering/causalize facts, no device state
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) fail(SC_ERR_INVALID_ARGUMENT, "bad device ordinal");
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(device), "cudaSetDevice");
  // one weight blob; each op's arrays 256-byte aligned
  const size_t nops = plan->prog.ops.size();
  plan->dops.assign(nops, DevOp{});
  std::vector<std::vector<float>> wtc(nops);
  for (size_t i = 0; i < nops; ++i) plan_tc(plan->prog, i, precision, plan->dops[i], wtc[i]);
  // fp32 plans: every tensor-core op outside a chain-eligible pair takes the 3xFP16 split
  if (precision == SC_PREC_FP32 && !split_tf32()) {
    std::vector<uint8_t> chained(nops, 0);
    {
      std::vector<DevOp> probe = plan->dops;
      find_chains(plan->prog, probe, wtc, false);
      for (size_t i = 0; i < nops; ++i)
        if (probe[i].chain >= 0) chained[i] = chained[static_cast<size_t>(probe[i].chain)] = 1;
    }
    for (size_t i = 0; i < nops; ++i)
      // (a LeakyReLU slope > 1 on the input stays on 3xTF32: the 3xFP16 transform applies the
      // pre-activation as max(x, a x), which is LeakyReLU only for a <= 1,
      // and scales rows by max |x| >= max |act(x)|)
      // (a tanh on the input stays there too: its 3xFP16 form would put a call per element into
      // the transform; no config uses it)
      if (plan->dops[i].kernel == KERNEL_TC && !chained[i] && plan->prog.ops[i].pre_act != ACT_TANH &&
          !(plan->prog.ops[i].pre_act == ACT_LRELU && std::fabs(plan->prog.ops[i].pre_alpha) > 1.f)) {
        plan->dops[i] = DevOp{};
        plan_tc(plan->prog, i, precision, plan->dops[i], wtc[i], true);
      }
  }
  if (!chain_disabled()) find_chains(plan->prog, plan->dops, wtc);
  // PQMF fast form: the factor arrays (S, C, class index as float) follow the op's blob slots
  std::vector<std::vector<float>> pqv(nops);
  for (size_t i = 0; i < nops; ++i) {
    const ConvOp& op = plan->prog.ops[i];
    DevOp& d = plan->dops[i];
    if (!op.pqmf || d.kernel != KERNEL_SIMT || pqmf_disabled() || op.gate || op.res_buf >= 0) continue;
    const BufferSpec& bi = plan->prog.bufs[op.in_buf];
    const BufferSpec& bo = plan->prog.bufs[op.out_buf];
    // one output row = M contiguous floats: an M-band frame (analysis) or M mono samples (synthesis)
    if (op.out_rstride != op.nout || op.nout != op.pq_M || bo.C != (op.pqmf == 1 ? op.pq_M : 1)) continue;
    if (op.pqmf == 1) {
      if (!pqmf_fast_shape(1, op.pq_M, op.pq_A, op.pq_B) || bi.C != 1 || op.row_step != op.pq_M || op.tap_step != 1)
        continue;
      d.kernel = KERNEL_PQMF_ANA;
    } else {
      if (!pqmf_fast_shape(2, op.pq_M, op.pq_A, op.pq_B, op.pq_period, op.pq_mirror) || op.row_step != 1 || op.tap_step != 1) continue;
      d.kernel = KERNEL_PQMF_SYN;
      d.pq_classes = op.pq_B;
    }
    // coefficients by value for the kernels' parameter bank: analysis S | Cm | bias[M],
    // synthesis R | s | bias[0] (kernels_pqmf.hpp PqmfCoef)
    d.pq_k.assign(sizeof(PqmfCoef) / sizeof(float), 0.f);
    if (op.pq_S.size() + op.pq_C.size() + op.bias.size() > d.pq_k.size()) {
      d.kernel = KERNEL_SIMT;
      continue;
    }
    if (op.pqmf == 1) {
      std::copy(op.pq_S.begin(), op.pq_S.end(), d.pq_k.begin());
      std::copy(op.pq_C.begin(), op.pq_C.end(), d.pq_k.begin() + op.pq_S.size());
      std::copy(op.bias.begin(), op.bias.end(), d.pq_k.begin() + op.pq_S.size() + op.pq_C.size());
    } else {
      std::copy(op.pq_C.begin(), op.pq_C.end(), d.pq_k.begin());
      std::copy(op.pq_S.begin(), op.pq_S.end(), d.pq_k.begin() + op.pq_C.size());
      if (!op.bias.empty()) d.pq_k[op.pq_C.size() + op.pq_S.size()] = op.bias[0];
    }
    auto& v = pqv[i];
    const size_t nS = round_up(static_cast<int64_t>(op.pq_S.size()), 64);
    const size_t nC = round_up(static_cast<int64_t>(op.pq_C.size()), 64);
    v.assign(nS + nC + op.pq_idx.size(), 0.f);
    std::copy(op.pq_S.begin(), op.pq_S.end(), v.begin());
    std::copy(op.pq_C.begin(), op.pq_C.end(), v.begin() + nS);
    for (size_t k = 0; k < op.pq_idx.size(); ++k) v[nS + nC + k] = static_cast<float>(op.pq_idx[k]);
  }
  int64_t total = 0;
  std::vector<int64_t> woff, boff, toff, qoff;
  for (size_t i = 0; i < nops; ++i) {
    const ConvOp& op = plan->prog.ops[i];
    woff.push_back(total);
    total += round_up(static_cast<int64_t>(op.w.size()), 64);
    boff.push_back(total);
    total += round_up(static_cast<int64_t>(op.bias.size()), 64);
    toff.push_back(total);
    total += round_up(static_cast<int64_t>(wtc[i].size()), 64);
    qoff.push_back(total);
    total += round_up(static_cast<int64_t>(pqv[i].size()), 64);
  }
  std::vector<float> host(static_cast<size_t>(std::max<int64_t>(total, 1)), 0.f);
  for (size_t i = 0; i < nops; ++i) {
    const ConvOp& op = plan->prog.ops[i];
    std::memcpy(host.data() + woff[i], op.w.data(), op.w.size() * sizeof(float));
    std::memcpy(host.data() + boff[i], op.bias.data(), op.bias.size() * sizeof(float));
    if (!wtc[i].empty()) std::memcpy(host.data() + toff[i], wtc[i].data(), wtc[i].size() * sizeof(float));
    if (!pqv[i].empty()) std::memcpy(host.data() + qoff[i], pqv[i].data(), pqv[i].size() * sizeof(float));
  }
  ck(cudaMalloc(&plan->wmem, host.size() * sizeof(float)), "cudaMalloc(weights)");
  ck(cudaMemcpy(plan->wmem, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice),
     "cudaMemcpy(weights)");
  for (size_t i = 0; i < nops; ++i) {
    DevOp& d = plan->dops[i];
    d.w = plan->wmem + woff[i];
    d.bias = plan->wmem + boff[i];
    if (d.kernel == KERNEL_PQMF_ANA || d.kernel == KERNEL_PQMF_SYN) {
      const ConvOp& op = plan->prog.ops[i];
      d.pq_S = plan->wmem + qoff[i];
      d.pq_C = d.pq_S + round_up(static_cast<int64_t>(op.pq_S.size()), 64);
      d.pq_idx = d.pq_C + round_up(static_cast<int64_t>(op.pq_C.size()), 64);
    }
    if (d.kernel == KERNEL_TC) {
      const ConvOp& op = plan->prog.ops[i];
      d.wtc = plan->wmem + toff[i];
      const uint64_t Kpad = static_cast<uint64_t>(d.taps_view) * d.cin_view_pad + d.k_chain;
      if (d.bf16)
        d.map_w = make_map3(d.wtc, Kpad, op.nout, 1, Kpad * 2, static_cast<uint64_t>(op.nout) * Kpad * 2, 32,
                            d.BN, 1, true);
      else if (d.f16)
        d.map_w = make_map3(d.wtc, Kpad, op.nout, 2, Kpad * 2, static_cast<uint64_t>(op.nout) * Kpad * 2, 32,
                            d.BN, 1, false, true);
      else
        d.map_w = make_map3(d.wtc, Kpad, op.nout, 2, Kpad * 4, static_cast<uint64_t>(op.nout) * Kpad * 4, 32,
                            d.BN, 1);
    }
  }
  // bf16 plans store a buffer as bf16 when every op touching it is a tensor-core op (the bf16
  // operands are rounded once, by the producer) — halves the activation traffic
  plan->buf_bf16.assign(plan->prog.bufs.size(), 0);
  if (precision == SC_PREC_BF16 && !bf16_store_disabled()) {
    const Program& pg = plan->prog;
    const bool skip32 = bf16_skip_fp32();
    for (size_t b = 0; b < pg.bufs.size(); ++b) {
      bool ok = pg.bufs[b].C % 8 == 0;
      bool touched = b == 0;
      for (size_t i = 0; i < nops && ok; ++i) {
        const ConvOp& op = pg.ops[i];
        const DevOp& d = plan->dops[i];
        bool rd = op.in_buf == static_cast<int>(b);
        for (const SumIn& si : op.sum_in) rd = rd || si.buf == static_cast<int>(b);
        const bool rs = op.res_buf == static_cast<int>(b);
        const bool wr = op.out_buf == static_cast<int>(b);
        if (!rd && !rs && !wr) continue;
        touched = true;
        if (d.kernel != KERNEL_TC) ok = false;
        if (rd && op.in_off % 8 != 0) ok = false;
        if (rs && op.res_off % 8 != 0) ok = false;
        if (skip32 && (rs || (wr && op.res_buf >= 0))) ok = false;
        if (wr && op.out_rstride % 8 != 0) ok = false;
      }
      plan->buf_bf16[b] = (ok && touched) ? 1 : 0;
    }
    // a residual epilogue reads and writes the staging tile in place: its residual and output
    // buffers must share the element type
    for (bool changed = true; changed;) {
      changed = false;
      for (const ConvOp& op : pg.ops)
        if (op.res_buf >= 0 && plan->buf_bf16[op.res_buf] != plan->buf_bf16[op.out_buf]) {
          plan->buf_bf16[op.res_buf] = plan->buf_bf16[op.out_buf] = 0;
          changed = true;
        }
    }
  }
  plan->desc = plan->prog.describe();
  ck(cudaSetDevice(prev), "cudaSetDevice");
  return plan;
}

// --------------------------------------------------------------------------- state
void State::evict_lru_plan() {
  auto victim = plans.begin();
  for (auto it = plans.begin(); it != plans.end(); ++it)
    if (it->second->last_use < victim->second->last_use) victim = it;
  // its graphs / carry table may still be in flight on some stream: wait for the device
  // (eviction only happens with ever-changing buffer geometries, never in steady state)
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize(evict)");
  for (auto& g : victim->second->graphs) {
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    if (g.second.graph) cudaGraphDestroy(g.second.graph);
  }
  if (victim->second->d_desc) cudaFree(victim->second->d_desc);
  plan_bytes -= victim->second->dev_bytes;
  plans.erase(victim);
}

State::~State() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  for (auto& kv : plans) {
    for (auto& g : kv.second->graphs) {
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
      if (g.second.graph) cudaGraphDestroy(g.second.graph);
    }
    if (kv.second->d_desc) cudaFree(kv.second->d_desc);
  }
  if (capture_stream) cudaStreamDestroy(capture_stream);
  for (int k = 0; k < 2; ++k) {
    if (io_in[k]) cudaFree(io_in[k]);
    if (io_out[k]) cudaFree(io_out[k]);
    if (io_in16[k]) cudaFree(io_in16[k]);
    if (io_out16[k]) cudaFree(io_out16[k]);
    if (ev_entry[k]) cudaEventDestroy(ev_entry[k]);
    if (ev_h2d[k]) cudaEventDestroy(ev_h2d[k]);
    if (ev_comp[k]) cudaEventDestroy(ev_comp[k]);
    if (ev_d2h[k]) cudaEventDestroy(ev_d2h[k]);
  }
  if (s_h2d) cudaStreamDestroy(s_h2d);
  if (s_comp) cudaStreamDestroy(s_comp);
  if (s_d2h) cudaStreamDestroy(s_d2h);
  if (mem) cudaFree(mem);
  if (d_desc) cudaFree(d_desc);
  if (d_ids) cudaFree(d_ids);
  cudaSetDevice(prev);
}

std::unique_ptr<State> make_state(const Plan* plan, int streams, int64_t max_frames) {
  const Program& pg = plan->prog;
  if (plan->device < 0) fail(SC_ERR_INVALID_ARGUMENT, "plan was created host-only (device -1)");
  if (streams < 1) fail(SC_ERR_INVALID_ARGUMENT, "n_streams must be >= 1");
  if (max_frames < 1) fail(SC_ERR_INVALID_ARGUMENT, "max_frames must be >= 1");
  if ((max_frames * pg.sink_rate.num) % pg.sink_rate.den != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "max_frames x sink rate is not an integer");
  if (max_frames % pg.ratio != 0 && pg.ratio % max_frames != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO,
         "max_frames " + std::to_string(max_frames) + " is neither a multiple nor a divisor of the compression ratio " +
             std::to_string(pg.ratio));
  auto st = std::make_unique<State>();
  st->plan = plan;
  st->streams = streams;
  st->max_frames = max_frames;
  // Buffers shorter than the compression ratio need phase state: a stride-S reader keeps up
  // to S-1 pending input frames (cache + S, still S-aligned) and the sink keeps a FIFO of up
  // to (ratio - 1) x sink-rate frames (the fixed output lag).
  st->phase_mode = max_frames % pg.ratio != 0;
  st->cache.clear();
  for (const BufferSpec& b : pg.bufs) st->cache.push_back(b.cache);
  if (st->phase_mode) {
    // every operand of a Sum (and a residual epilogue) must receive its frames in lockstep with
    // the other operands; a branch that changes rate internally does not under phase state
    std::vector<int64_t> n(pg.bufs.size(), 0);
    for (int64_t k = 0; k < 2 * pg.ratio; ++k) {
      n[0] += 1;
      for (const ConvOp& op : pg.ops) {
        const int64_t nin = n[op.in_buf];
        n[op.out_buf] = op.convt ? nin * op.r : (op.S > 1 ? (nin / op.S) * op.phases : nin);
        bool ok = op.res_buf < 0 || n[op.res_buf] == n[op.out_buf];
        for (const SumIn& si : op.sum_in) ok = ok && n[si.buf] == nin;
        if (!ok)
          fail(SC_ERR_UNSUPPORTED_FORMAT, "buffers shorter than the compression ratio with a Sum whose operands change rate "
                                          "inside the branch (" + op.name + ")");
      }
    }
    for (const ConvOp& op : pg.ops)
      if (!op.convt && op.S > 1) st->cache[op.in_buf] = std::max(st->cache[op.in_buf], pg.bufs[op.in_buf].cache + op.S);
    st->cache[pg.sink_buf] += (pg.ratio - 1) * pg.sink_rate.num / pg.sink_rate.den;
  }
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  // strip length: k calls' frames after the cache (phase mode keeps k = 1: bursts vary).
  // Strips pay off when the carry moves a lot of bytes (many streams x large caches); small
  // states keep k = 1 (one CallPlan / graph per buffer length).
  {
    int64_t cache_floats = 0;
    for (size_t i = 0; i < pg.bufs.size(); ++i) cache_floats += st->cache[i] * plan->fw(i);
    const bool big = cache_floats * 4 * static_cast<int64_t>(streams) >= (int64_t{256} << 20);
    const char* e = std::getenv("SC_STRIP_K");
    st->strip_k = st->phase_mode ? 1 : std::max(1, e ? std::atoi(e) : (big ? 4 : 1));
  }
  {
    const char* e = std::getenv("SC_REDZONE");
    if (e && e[0] != '0') {
      st->rz_stream = 64;
      st->rz_gap = 4096;
    }
  }
  std::vector<int64_t> off;
  for (;;) {
    int64_t total = 0;
    off.clear();
    st->buf_sstride.clear();
    st->rz_used.clear();
    st->cache_bytes_per_stream = 0;
    for (size_t i = 0; i < pg.bufs.size(); ++i) {
      const BufferSpec& b = pg.bufs[i];
      // a call may deliver up to (F + ratio) input samples' worth of frames (phase bursts)
      const int64_t T = ((max_frames + pg.ratio) * b.rate.num + b.rate.den - 1) / b.rate.den;
      const int64_t used = (st->cache[i] + st->strip_k * T + b.tail) * plan->fw(i);
      const int64_t sstride = round_up(used + st->rz_stream, 32);
      st->buf_sstride.push_back(sstride);
      st->rz_used.push_back(used);
      total += st->rz_gap;
      off.push_back(total);
      total += round_up(sstride * streams, 64);
      st->cache_bytes_per_stream += st->cache[i] * plan->fw(i) * 4;
    }
    total += st->rz_gap;
    st->mem_bytes = total * 4;
    const cudaError_t e = cudaMalloc(&st->mem, std::max<int64_t>(st->mem_bytes, 256));
    if (e == cudaSuccess) break;
    cudaGetLastError();
    if (st->strip_k == 1) ck(e, "cudaMalloc(state)");
    st->strip_k /= 2;  // not enough memory for this strip length: halve it (k = 1: carry every call)
  }
  ck(cudaMemset(st->mem, 0, std::max<int64_t>(st->mem_bytes, 256)), "cudaMemset(state)");
  for (size_t i = 0; i < pg.bufs.size(); ++i) st->buf_base.push_back(st->mem + off[i]);
  if (st->rz_stream > 0) {
    st->redzone_fill(nullptr);
    ck(cudaDeviceSynchronize(), "redzone fill");
  }
  // reset table: buffers with a cache
  std::vector<BufDesc> desc;
  int64_t ritems = 0;
  for (size_t i = 0; i < pg.bufs.size(); ++i) {
    const BufferSpec& b = pg.bufs[i];
    if (st->cache[i] == 0) continue;
    BufDesc d{};
    d.base = st->buf_base[i];
    d.sstride = st->buf_sstride[i];
    d.ritem0 = ritems;
    d.C = plan->fw(i);
    d.cache = static_cast<int>(st->cache[i]);
    ritems += plan->fw(i);
    desc.push_back(d);
  }
  if (desc.size() > 64) fail(SC_ERR_UNSUPPORTED_FORMAT, "more than 64 cached buffers");
  st->n_desc = static_cast<int>(desc.size());
  st->reset_items = ritems;
  st->reset_desc = desc;
  st->pos.assign(pg.bufs.size(), 0);
  st->carry_slot = !desc.empty();
  if (!desc.empty()) {
    ck(cudaMalloc(&st->d_desc, desc.size() * sizeof(BufDesc)), "cudaMalloc(desc)");
    ck(cudaMemcpy(st->d_desc, desc.data(), desc.size() * sizeof(BufDesc), cudaMemcpyHostToDevice),
       "cudaMemcpy(desc)");
  }
  ck(cudaMalloc(&st->d_ids, sizeof(int) * streams), "cudaMalloc(ids)");
  ck(cudaStreamCreateWithFlags(&st->capture_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  st->N.assign(pg.bufs.size(), 0);
  ck(cudaSetDevice(prev), "cudaSetDevice");
  return st;
}

// Cumulative frames per buffer after one more call of F input samples: every op emits what
// its accumulated input allows (stride S: floor(N_in / S); ConvT r: r N_in; else N_in).
std::vector<int64_t> State::next_counts(int64_t F) const {
  const Program& pg = plan->prog;
  std::vector<int64_t> n(N);
  n[0] = N[0] + F;
  for (const ConvOp& op : pg.ops) {
    const int64_t nin = n[op.in_buf];
    n[op.out_buf] = op.convt ? nin * op.r : (op.S > 1 ? (nin / op.S) * op.phases : nin);
  }
  return n;
}

CallPlan& State::call_plan(int64_t F) {
  const Program& pg = plan->prog;
  const std::vector<int64_t> n = next_counts(F);
  const int64_t Fs = F * pg.sink_rate.num / pg.sink_rate.den;
  const int sb = pg.sink_buf;
  const int64_t D_ = (D < 0) ? lag_for(F) : D;
  const int64_t row = (E - D_) - N[sb] + cache[sb];
  if (E + Fs - D_ > n[sb] || row < 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO,
         "buffer length " + std::to_string(F) + " cannot continue this stream at lag " + std::to_string(D_) +
             " (use one constant length below the compression ratio " + std::to_string(pg.ratio) + ")");
  // strip positions: a buffer whose cache + new frames would run past its strip wraps first
  // (its cache moves to the strip start: the carry, once per strip_k calls)
  std::vector<int64_t> pw(pos);
  for (size_t b = 0; b < n.size(); ++b) {
    const int64_t cap = buf_sstride[b] / plan->fw(b);
    if (pos[b] + cache[b] + (n[b] - N[b]) > cap) pw[b] = 0;
  }
  std::vector<int64_t> key;
  key.push_back(F);
  key.push_back(row);
  for (size_t b = 0; b < n.size(); ++b) key.push_back(n[b] - N[b]);
  for (const ConvOp& op : pg.ops) key.push_back(op.S > 1 && !op.convt ? N[op.in_buf] % op.S : 0);
  for (size_t b = 0; b < n.size(); ++b) key.push_back(pos[b]);
  auto it = plans.find(key);
  if (it != plans.end()) {
    it->second->last_use = ++plan_clock;
    return *it->second;
  }
  if (plans.size() >= kMaxCallPlans) evict_lru_plan();

  auto cp = std::make_unique<CallPlan>();
  cp->pos = pw;
  for (size_t b = 0; b < n.size(); ++b) cp->base.push_back(buf_base[b] + pw[b] * plan->fw(b));
  cp->F = F;
  cp->egress_row = row - pg.sink_delay;  // a Delay in front of the Sink (cache >= delay)
  cp->egress_T = Fs;
  for (size_t b = 0; b < n.size(); ++b) cp->T.push_back(n[b] - N[b]);
  for (const ConvOp& op : pg.ops) {
    cp->pend.push_back(op.S > 1 && !op.convt ? N[op.in_buf] % op.S : 0);
    cp->t_out.push_back(op.convt ? cp->T[op.in_buf] : cp->T[op.out_buf] / op.phases);
  }
  for (size_t b = 0; b < pg.bufs.size(); ++b)
    if (cache[b] > static_cast<int64_t>(buf_sstride[b] / plan->fw(b)) - cp->T[b])
      fail(SC_ERR_INVALID_ARGUMENT, "buffer length exceeds max_frames");
  // carry table (runs first): wrapped buffers move their cache from row pos to the strip start
  std::vector<BufDesc> desc;
  int64_t items = 0;
  for (size_t i = 0; i < pg.bufs.size(); ++i) {
    const BufferSpec& b = pg.bufs[i];
    if (cache[i] == 0 || pw[i] == pos[i]) continue;
    BufDesc d{};
    d.base = buf_base[i];
    d.sstride = buf_sstride[i];
    d.item0 = items;
    d.C = plan->fw(i);
    d.cache = static_cast<int>(cache[i]);
    d.t = static_cast<int>(pos[i]);
    items += static_cast<int64_t>(streams) * ((d.C % 4 == 0) ? d.C / 4 : d.C);  // float4 groups
    desc.push_back(d);
  }
  if (desc.size() > 64) fail(SC_ERR_UNSUPPORTED_FORMAT, "more than 64 cached buffers");
  cp->n_desc = static_cast<int>(desc.size());
  cp->carry_items = items;
  cp->n_launch = 2 + (desc.empty() ? 0 : 1);
  for (int64_t t : cp->t_out) cp->n_launch += t > 0 ? 1 : 0;
  if (!desc.empty()) {
    ck(cudaMalloc(&cp->d_desc, desc.size() * sizeof(BufDesc)), "cudaMalloc(desc)");
    cp->dev_bytes = static_cast<int64_t>(desc.size() * sizeof(BufDesc));
    plan_bytes += cp->dev_bytes;
    ck(cudaMemcpy(cp->d_desc, desc.data(), desc.size() * sizeof(BufDesc), cudaMemcpyHostToDevice),
       "cudaMemcpy(desc)");
  }
  // tensor-core launches (tensor maps depend on the tile geometry and the pending offset)
  cp->tc.resize(pg.ops.size());
  for (size_t i = 0; i < pg.ops.size(); ++i) {
    const DevOp& d = plan->dops[i];
    if (d.kernel != KERNEL_TC || cp->t_out[i] == 0) continue;
    const ConvOp& op = pg.ops[i];
    const BufferSpec& bi = pg.bufs[op.in_buf];
    const ConvParams c = conv_params(i, *cp);
    const int S = d.view_S;
    // window start frame; super-rows are anchored at base_off so that it is S-aligned
    const int64_t f0 = c.in_f0;
    const int64_t base_off = f0 % S;
    const uint64_t bufC_view = static_cast<uint64_t>(bi.C) * S;
    const int64_t frames_avail = buf_sstride[op.in_buf] / plan->fw(op.in_buf) - cp->pos[op.in_buf] - base_off;
    const bool a_bf = plan->buf_bf16[op.in_buf] != 0;
    const bool o_bf = plan->buf_bf16[op.out_buf] != 0;
    const bool r_bf = op.res_buf >= 0 && plan->buf_bf16[op.res_buf] != 0;
    const uint64_t aes = a_bf ? 2 : 4, oes = o_bf ? 2 : 4, res_es = r_bf ? 2 : 4;
    const uint64_t rows_view = static_cast<uint64_t>(frames_avail / S);
    TcParams& p = cp->tc[i].p;
    p.BN = d.BN;
    p.bf16 = d.bf16 ? 1 : 0;
    const int t_out = c.t_out;
    if (t_out >= 128) {
      p.R = 128;
      p.G = 1;
      p.tiles_per_stream = (t_out + 127) / 128;
      p.m_tiles = p.tiles_per_stream * streams;
    } else {
      p.R = t_out;
      p.G = std::min(128 / t_out, streams);
      p.tiles_per_stream = 1;
      p.m_tiles = (streams + p.G - 1) / p.G;
    }
    // few output tiles (deep layers at small stream counts, e.g. 1 frame x 128 streams): halve
    // the N tile towards a grid that covers the SMs.  The K order does not depend on BN, so results
    // are bit-identical to the full-width tile (buffer-partition / stream-count invariance).
    if (!c.gate && plan->dops[i].chain < 0 && !small_bn_disabled()) {
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
      // ... but only while the narrower tiles still fit one wave: the per-slab cost of these tiles
      // is mostly the transform of the input rows, which does not shrink with BN, so a second wave
      // of narrow tiles costs more than the idle SMs it fills (cfg5 at 2048 streams: 1.81 -> 1.70
      // ms per step; at 128 streams narrowing still gains 10-25%)
      while (p.BN > 32 && c.nout % (p.BN / 2) == 0 &&
             static_cast<int64_t>(p.m_tiles) * ((c.nout + p.BN / 2 - 1) / (p.BN / 2)) <= sms)
        p.BN /= 2;
    }
    if (p.BN != d.BN) {  // this call's weight boxes: BN rows
      const uint64_t Kpad = static_cast<uint64_t>(d.taps_view) * d.cin_view_pad + d.k_chain;
      const int es = (d.bf16 || d.f16) ? 2 : 4;
      cp->tc[i].map_w = make_map3(d.wtc, Kpad, op.nout, d.bf16 ? 1 : 2, Kpad * es,
                                  static_cast<uint64_t>(op.nout) * Kpad * es, 32, p.BN, 1, d.bf16, d.f16);
      cp->tc[i].own_w = true;
    }
    p.cblocks = d.cin_view_pad / 32;
    p.n_kblocks = d.taps_view * p.cblocks;
    p.a_c0 = S > 1 ? 0 : op.in_off;
    p.a_row0 = static_cast<int>((f0 - base_off) / S);
    p.a_tap_rows = d.tap_rows;
    // window mode (fp32, BN <= 64, one stream per tile): the transform splits each input row
    // once per 32-channel block and every tap's MMAs read it at a row offset
    p.halo = (d.taps_view - 1) * d.tap_rows;
    // a layer that may run in window mode for some call geometry accumulates in the window
    // order in every mode (bit-identity across partitions); a static property of the layer
    p.cbmaj = ((d.bf16 || d.f16 || d.BN <= 64) && d.taps_view > 1) ? 1 : 0;
    p.win = ((d.bf16 || d.f16 || d.BN <= 64) && p.G == 1 && d.taps_view > 1 && p.R + p.halo <= ((d.bf16 && (d.BN < 128 || plan->buf_bf16[op.in_buf])) ? 192 : 144) &&
             !win_disabled() && !(plan->dops[i].chain >= 0 && !d.bf16)) ? 1 : 0;
    // ... and the whole weight (hi + lo, every K-slab) resident when it fits 112 KB
    p.wres = (p.win && !d.bf16 && static_cast<int64_t>(d.taps_view) * (d.cin_view_pad / 32) * 2 * p.BN * 32 * (d.f16 ? 2 : 4) <=
                                        (d.f16 ? 56 : 112) * 1024 &&
              op.nout == p.BN) ? 1 : 0;
    p.f16 = d.f16 ? 1 : 0;
    p.f16_sw = d.f16_sw;
    p.awin = (d.f16 && !p.win && p.cbmaj && d.taps_view > 1 && (p.R + p.halo) * p.G <= 192 && !awin_disabled()) ? 1 : 0;
    p.pre_act = c.pre_act;
    p.pre_alpha = c.pre_alpha;
    p.post_act = c.post_act;
    p.post_alpha = c.post_alpha;
    p.gate = c.gate;
    p.nout = c.nout;
    p.t_out = t_out;
    p.streams = streams;
    p.bias = c.bias;
    p.out = c.out;
    p.out_sstride = c.out_sstride;
    p.out_base = c.out_base;
    p.out_rstride = c.out_rstride;
    p.res = c.res;
    p.res_sstride = c.res_sstride;
    p.res_fstride = c.res_fstride;
    p.res_off = c.res_off;
    p.res_f0 = c.res_f0;
    p.res_act = c.res_act;
    p.res_alpha = c.res_alpha;
    {
      const char* dbg = std::getenv("SC_TC_DEBUG");
      p.debug = dbg ? std::atoi(dbg) : 0;
      const char* tr = std::getenv("SC_TC_TRACE_OP");
      if (tr && std::atoi(tr) == static_cast<int>(i)) p.debug |= 32;
    }
    p.a_bf = a_bf ? 1 : 0;
    p.o_bf = o_bf ? 1 : 0;
    p.r_bf = r_bf ? 1 : 0;
    // word (4-byte) offsets into the buffers: a bf16 buffer packs two elements per word
    cp->tc[i].map_a = make_map3(cp->base[op.in_buf] + base_off * plan->fw(op.in_buf), bufC_view, rows_view, streams,
                                bufC_view * aes, static_cast<uint64_t>(buf_sstride[op.in_buf]) * 4, 32,
                                static_cast<uint32_t>(p.R + ((p.win || p.awin) ? p.halo : 0)), static_cast<uint32_t>(p.G), a_bf);
    // output rows start at the cache end; rows >= t_out and streams >= n_streams are clipped by TMA
    cp->tc[i].map_out = make_map3(c.out + cache[op.out_buf] * plan->fw(op.out_buf), static_cast<uint64_t>(c.out_rstride),
                                  static_cast<uint64_t>(t_out), streams, static_cast<uint64_t>(c.out_rstride) * oes,
                                  static_cast<uint64_t>(c.out_sstride) * 4, 32, static_cast<uint32_t>(p.R),
                                  static_cast<uint32_t>(p.G), o_bf);
    if (c.res) {
      cp->tc[i].map_res = make_map3(c.res + static_cast<int64_t>(c.res_f0) * plan->fw(op.res_buf),
                                    static_cast<uint64_t>(c.res_fstride), static_cast<uint64_t>(t_out), streams,
                                    static_cast<uint64_t>(c.res_fstride) * res_es,
                                    static_cast<uint64_t>(c.res_sstride) * 4, 32, static_cast<uint32_t>(p.R),
                                    static_cast<uint32_t>(p.G), r_bf);
    } else {
      cp->tc[i].map_res = cp->tc[i].map_out;  // unused
    }
  }
  // chained 1x1 convs (find_chains): one launch computes both when this call gives them the
  // same tile geometry; the second conv's epilogue (bias, act, residual, output) moves over
  cp->chained.assign(pg.ops.size(), -1);
  for (size_t i = 0; i < pg.ops.size(); ++i) {
    const int j = plan->dops[i].chain;
    if (j < 0 || cp->t_out[i] == 0 || cp->t_out[j] != cp->t_out[i]) continue;
    TcParams& a = cp->tc[i].p;
    const TcParams& b = cp->tc[j].p;
    if ((a.win && !a.bf16) || b.win || a.R != b.R || a.G != b.G || a.m_tiles != b.m_tiles) continue;
    a.chain = 128 / 32;
    a.chain_one = plan->dops[i].chain_one || a.bf16;  // bf16: K = 128 is one CK = 4 chunk anyway
    a.mid_bf = plan->buf_bf16[pg.ops[i].out_buf];
    a.o_bf = b.o_bf;
    a.r_bf = b.r_bf;
    a.bias2 = b.bias;
    a.mid_act1 = a.post_act;
    a.mid_alpha1 = a.post_alpha;
    a.mid_act2 = b.pre_act;
    a.mid_alpha2 = b.pre_alpha;
    a.post_act = b.post_act;
    a.post_alpha = b.post_alpha;
    a.gate = b.gate;
    a.nout = b.nout;
    a.out = b.out;
    a.out_sstride = b.out_sstride;
    a.out_base = b.out_base;
    a.out_rstride = b.out_rstride;
    a.res = b.res;
    a.res_sstride = b.res_sstride;
    a.res_fstride = b.res_fstride;
    a.res_off = b.res_off;
    a.res_f0 = b.res_f0;
    a.res_act = b.res_act;
    a.res_alpha = b.res_alpha;
    cp->tc[i].map_out = cp->tc[j].map_out;
    cp->tc[i].map_res = cp->tc[j].map_res;
    cp->t_out[j] = 0;  // not launched: op i's launch writes its output
    cp->chained[i] = j;
    cp->n_launch -= 1;
  }
  // fused mono I/O: the PQMF analysis reads the caller's input itself (its window's cached rows
  // from the strip, the new rows from the caller, and it writes the last cache rows back as the
  // next call's cache), the PQMF synthesis writes the caller's output — no ingest / egress
  // launch and no strip round trip for the mono signal (C = 1: [stream][1][T] is the frame-major
  // layout already).  Only when the geometry is the plain one; else the separate kernels run.
  if (!io_fuse_disabled()) {
    int reader = -1, readers = 0, writer = -1, writers = 0;
    for (size_t i = 0; i < pg.ops.size(); ++i) {
      const ConvOp& op = pg.ops[i];
      if (op.in_buf == 0) reader = static_cast<int>(i), ++readers;
      if (op.res_buf == 0) readers += 2;
      for (const SumIn& si : op.sum_in) readers += si.buf == 0 ? 2 : 0;
      if (op.out_buf == pg.sink_buf) writer = static_cast<int>(i), ++writers;
      if (op.res_buf == pg.sink_buf || op.in_buf == pg.sink_buf) writers += 2;
      for (const SumIn& si : op.sum_in) writers += si.buf == pg.sink_buf ? 2 : 0;
    }
    if (readers == 1 && plan->dops[reader].kernel == KERNEL_PQMF_ANA && pg.in_C == 1 && !plan->buf_bf16[0] &&
        cp->t_out[reader] > 0) {
      const ConvParams c = conv_params(reader, *cp);
      const int64_t last_i0 = ((c.t_out - 1) / 128) * 128;
      if (F >= cache[0] && c.in_f0 + 16 * static_cast<int64_t>(c.t_out) + kPqmfLook == cache[0] + F &&
          c.in_f0 + 16 * last_i0 <= F && c.in_f0 >= 0)
        cp->fuse_in = reader;
    }
    if (writers == 1 && plan->dops[writer].kernel == KERNEL_PQMF_SYN && pg.sink_C == 1 && pg.sink_off == 0 &&
        pg.sink_act == ACT_ID && cache[sb] == 0 && !plan->buf_bf16[sb] && cp->t_out[writer] > 0 &&
        cp->egress_row == 0 && cp->egress_T == 16 * cp->t_out[writer] && pg.bufs[sb].C == 1)
      cp->fuse_out = writer;
    cp->n_launch -= (cp->fuse_in >= 0 ? 1 : 0) + (cp->fuse_out >= 0 ? 1 : 0);
  }
  cp->last_use = ++plan_clock;
  return *plans.emplace(key, std::move(cp)).first->second;
}

ConvParams State::conv_params(size_t i, const CallPlan& cp) const {
  const Program& pg = plan->prog;
  const ConvOp& op = pg.ops[i];
  const BufferSpec& bi = pg.bufs[op.in_buf];
  const BufferSpec& bo = pg.bufs[op.out_buf];
  ConvParams p{};
  p.in = cp.base[op.in_buf];
  p.in_sstride = buf_sstride[op.in_buf];
  p.in_fstride = bi.C;
  p.in_off = op.in_off;
  p.cin = op.cin;
  p.in_f0 = static_cast<int>(cache[op.in_buf] - op.look - cp.pend[i]);
  p.row_step = op.row_step;
  p.tap_step = op.tap_step;
  p.taps = op.taps;
  p.w = plan->dops[i].w;
  p.bias = plan->dops[i].bias;
  p.nout = op.nout;
  p.out = cp.base[op.out_buf];
  p.out_sstride = buf_sstride[op.out_buf];
  p.out_base = cache[op.out_buf] * bo.C;
  p.out_rstride = op.out_rstride;
  p.t_out = static_cast<int>(cp.t_out[i]);
  p.streams = streams;
  p.pre_act = op.pre_act;
  p.pre_alpha = op.pre_alpha;
  p.post_act = op.post_act;
  p.post_alpha = op.post_alpha;
  p.gate = op.gate ? 1 : 0;
  if (op.res_buf >= 0) {
    const BufferSpec& br = pg.bufs[op.res_buf];
    p.res = cp.base[op.res_buf];
    p.res_sstride = buf_sstride[op.res_buf];
    p.res_fstride = br.C;
    p.res_off = op.res_off;
    p.res_f0 = static_cast<int>(cache[op.res_buf] - op.res_delay);
    p.res_act = op.res_act;
    p.res_alpha = op.res_alpha;
  }
  return p;
}

PqmfParams State::pqmf_params(size_t i, const CallPlan& cp) const {
  const ConvParams c = conv_params(i, cp);
  const DevOp& d = plan->dops[i];
  PqmfParams p{};
  p.in = c.in;
  p.in_sstride = c.in_sstride;
  p.in_fstride = c.in_fstride;
  p.in_off = c.in_off;
  p.in_f0 = c.in_f0;
  p.S = d.pq_S;
  p.C = d.pq_C;
  p.idx = d.pq_idx;
  p.bias = c.bias;
  p.nclass = d.pq_classes;
  p.period = plan->prog.ops[i].pq_period;
  p.mirror = plan->prog.ops[i].pq_mirror;
  p.out = c.out;
  p.out_sstride = c.out_sstride;
  p.out_base = c.out_base;
  p.t_out = c.t_out;
  p.streams = c.streams;
  p.pre_act = c.pre_act;
  p.pre_alpha = c.pre_alpha;
  p.post_act = c.post_act;
  p.post_alpha = c.post_alpha;
  return p;
}

PqmfParams State::pqmf_io_params(size_t i, const CallPlan& cp, const float* in, float* out) const {
  PqmfParams p = pqmf_params(i, cp);
  if (static_cast<int>(i) == cp.fuse_in) {
    p.xin = in;
    p.strip = cp.base[0];
    p.xin_T = static_cast<int>(cp.F);
    p.cache0 = static_cast<int>(cache[0]);
  }
  if (static_cast<int>(i) == cp.fuse_out) {
    p.out = out;
    p.out_sstride = cp.egress_T;
    p.out_base = 0;
  }
  return p;
}

SumParams State::sum_params(size_t i, const CallPlan& cp) const {
  const Program& pg = plan->prog;
  const ConvOp& op = pg.ops[i];
  SumParams p{};
  p.n_in = static_cast<int>(op.sum_in.size());
  for (int q = 0; q < p.n_in; ++q) {
    const SumIn& si = op.sum_in[q];
    p.in[q] = cp.base[si.buf];
    p.in_sstride[q] = buf_sstride[si.buf];
    p.in_fstride[q] = pg.bufs[si.buf].C;
    p.in_off[q] = si.off;
    p.in_f0[q] = static_cast<int>(cache[si.buf] - si.delay);
    p.act[q] = si.act;
    p.alpha[q] = si.alpha;
  }
  p.out = cp.base[op.out_buf];
  p.out_sstride = buf_sstride[op.out_buf];
  p.out_base = cache[op.out_buf] * pg.bufs[op.out_buf].C;
  p.C = op.nout;
  p.t_out = static_cast<int>(cp.t_out[i]);
  p.streams = streams;
  p.post_act = op.post_act;
  p.post_alpha = op.post_alpha;
  return p;
}

// NVTX ranges (SC_NVTX=1): one per process call, and one per launch in eager mode (graph
// replays have no host-side launches to mark) — layer names as in sc_launch_name
bool nvtx_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SC_NVTX");
    return e && e[0] != '0';
  }();
  return on;
}

struct NvtxRange {
  bool on;
  NvtxRange(bool enabled, const std::string& name) : on(enabled) {
    if (on) nvtxRangePushA(name.c_str());
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

IngestArgs State::ingest_args(const float* in, const CallPlan& cp) const {
  const Program& pg = plan->prog;
  IngestArgs a{};
  a.in = in;
  a.buf = cp.base[0];
  a.bf = plan->buf_bf16[0];
  a.sstride = buf_sstride[0];
  a.C = pg.in_C;
  a.T = static_cast<int>(cp.F);
  a.cache = static_cast<int>(cache[0]);
  a.streams = streams;
  return a;
}

EgressArgs State::egress_args(float* out, const CallPlan& cp) const {
  const Program& pg = plan->prog;
  const BufferSpec& b = pg.bufs[pg.sink_buf];
  EgressArgs a{};
  a.buf = cp.base[pg.sink_buf];
  a.bf = plan->buf_bf16[pg.sink_buf];
  a.sstride = buf_sstride[pg.sink_buf];
  a.fstride = b.C;
  a.off = pg.sink_off;
  a.C = pg.sink_C;
  a.T = static_cast<int>(cp.egress_T);
  a.cache = static_cast<int>(cp.egress_row);
  a.streams = streams;
  a.act = pg.sink_act;
  a.alpha = pg.sink_alpha;
  a.out = out;
  return a;
}

// RAII: make the plan's device current (call_plan allocates the carry table and encodes tensor
// maps on it) and restore the caller's device on every exit path, exceptions included.
struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    ck(cudaGetDevice(&prev), "cudaGetDevice");
    ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

int State::launches(int64_t F) {
  check_frames(F);
  DeviceScope dev(plan->device);
  CallPlan& cp = call_plan(F);
  int n = (cp.fuse_in < 0 ? 1 : 0) + (cp.fuse_out < 0 ? 1 : 0) + (carry_slot ? 1 : 0);
  for (int64_t t : cp.t_out) n += t > 0 ? 1 : 0;
  return n;
}

std::string State::launch_name(int64_t F, int i) {
  check_frames(F);
  DeviceScope dev(plan->device);
  CallPlan& cp = call_plan(F);
  int k = 0;
  if (carry_slot && i == k++) return "carry";
  if (cp.fuse_in < 0 && i == k++) return "ingest";
  for (size_t j = 0; j < plan->prog.ops.size(); ++j) {
    if (cp.t_out[j] == 0) continue;
    if (i == k++) {
      const ConvOp& op = plan->prog.ops[j];
      const DevOp& d = plan->dops[j];
      const int jc = cp.chained.empty() ? -1 : cp.chained[j];
      if (jc >= 0)
        return "op" + std::to_string(j) + "+" + std::to_string(jc) + " " + op.name + " + " +
               plan->prog.ops[jc].name + (plan->dops[j].bf16 ? " [tc-bf16]" : " [tc]");
      return "op" + std::to_string(j) + " " + op.name + " [" +
             (d.kernel == KERNEL_TC ? (d.bf16 ? "tc-bf16" : d.f16 ? "tc-3xf16" : "tc")
              : d.kernel == KERNEL_SIMT ? "simt" : d.kernel == KERNEL_SUM ? "simt-sum"
              : static_cast<int>(j) == cp.fuse_in ? "pqmf+input" : static_cast<int>(j) == cp.fuse_out ? "pqmf+output" : "pqmf") + "]";
    }
  }
  if (cp.fuse_out < 0 && i == k++) return "egress";
  return "";
}

void State::enqueue(const float* in, float* out, CallPlan& cp, cudaStream_t s, cudaEvent_t* ev) {
  int e = 0;
  if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  if (carry_slot) {  // wrapped buffers first move their cache to the strip start
    if (cp.n_desc > 0) launch_carry(cp.d_desc, cp.n_desc, streams, cp.carry_items, s);
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
  if (cp.fuse_in < 0) {
    launch_ingest(ingest_args(in, cp), s);
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
  for (size_t i = 0; i < plan->prog.ops.size(); ++i) {
    if (cp.t_out[i] == 0) continue;
    NvtxRange op_range(ev == nullptr && nvtx_enabled() && !capturing, "op" + std::to_string(i) + " " + plan->prog.ops[i].name);
    if (plan->dops[i].kernel == KERNEL_TC) {
      const TcLaunch& t = cp.tc[i];
      launch_conv_tc(t.map_a, t.own_w ? t.map_w : plan->dops[i].map_w, t.map_out, t.map_res, t.p, s);
    } else if (plan->dops[i].kernel == KERNEL_SUM) {
      launch_sum(sum_params(i, cp), s);
    } else if (plan->dops[i].kernel == KERNEL_PQMF_ANA || plan->dops[i].kernel == KERNEL_PQMF_SYN) {
      launch_pqmf(plan->dops[i].kernel == KERNEL_PQMF_ANA ? 1 : 2, pqmf_io_params(i, cp, in, out),
                  *reinterpret_cast<const PqmfCoef*>(plan->dops[i].pq_k.data()), s);
    } else {
      launch_conv_simt(conv_params(i, cp), s);
    }
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
  if (cp.fuse_out < 0) {
    launch_egress(egress_args(out, cp), s);
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
}

void State::check_frames(int64_t F) const {
  const Program& pg = plan->prog;
  if (F <= 0) fail(SC_ERR_INVALID_ARGUMENT, "frames must be positive");
  if ((F * pg.sink_rate.num) % pg.sink_rate.den != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO,
         "buffer length " + std::to_string(F) + " times the sink rate is not an integer");
  if (F % pg.ratio != 0 && (!phase_mode || pg.ratio % F != 0))
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "buffer length " + std::to_string(F) +
                                                  " is neither a multiple nor a divisor of the compression ratio " +
                                                  std::to_string(pg.ratio));
  if (F > max_frames)
    fail(SC_ERR_INVALID_ARGUMENT, "buffer length " + std::to_string(F) + " exceeds max_frames " +
                                      std::to_string(max_frames));
}

void State::profile(const float* in, float* out, int64_t F, int steps, float* ms, cudaStream_t s) {
  check_frames(F);
  if (steps < 1) fail(SC_ERR_INVALID_ARGUMENT, "steps must be >= 1");
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  const int n = launches(F);  // the layout (the carry slot is present whenever the state has caches)
  for (int i = 0; i < n; ++i) ms[i] = 0.f;
  std::vector<cudaEvent_t> ev(static_cast<size_t>(n + 1) * steps);
  for (auto& e : ev) ck(cudaEventCreate(&e), "EventCreate");
  int done = 0;
  for (int k = 0; k < steps; ++k) {
    CallPlan& cp = call_plan(F);
    const bool same = launches(F) == n;
    enqueue(in, out, cp, s, same ? ev.data() + static_cast<size_t>(k) * (n + 1) : nullptr);
    launched += cp.n_launch;
    advance(F, cp);
    if (same) ++done;
  }
  ck(cudaGetLastError(), "launch");
  ck(cudaStreamSynchronize(s), "StreamSynchronize");
  for (int k = 0; k < steps; ++k) {
    for (int i = 0; i < n; ++i) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev[static_cast<size_t>(k) * (n + 1) + i],
                               ev[static_cast<size_t>(k) * (n + 1) + i + 1]) == cudaSuccess && done > 0)
        ms[i] += t / done;
    }
  }
  cudaGetLastError();  // events of skipped steps were never recorded
  for (auto& e : ev) cudaEventDestroy(e);
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

void State::process(const float* in, float* out, int64_t F, cudaStream_t s) {
  check_frames(F);
  if (!in || !out) fail(SC_ERR_INVALID_ARGUMENT, "null I/O pointer");
  NvtxRange call_range(nvtx_enabled(), "sc_process F=" + std::to_string(F) + " streams=" + std::to_string(streams));
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  CallPlan& cp = call_plan(F);
  if (!use_graphs) {
    enqueue(in, out, cp, s, nullptr);
    ck(cudaGetLastError(), "launch");
    launched += cp.n_launch;
  } else {
    const auto key = std::make_pair(in, out);
    auto it = cp.graphs.find(key);
    if (it == cp.graphs.end()) {
      // One graph per CallPlan, re-targeted (ingest / egress kernel-node params) when the I/O
      // pointers change: a capture happens once per CallPlan (the strip cycle's few plans are
      // all met within the first calls), never again in steady state.
      GraphEntry g;
      if (cp.graphs.size() >= static_cast<size_t>(graphs_per_plan())) {
        auto lru = cp.graphs.begin();
        for (auto jt = cp.graphs.begin(); jt != cp.graphs.end(); ++jt)
          if (jt->second.last_use < lru->second.last_use) lru = jt;
        // the ingest / egress kernels (wide or general) are picked per I/O pointer at launch: a
        // graph captured with the other one cannot be re-targeted — drop it and capture anew
        const bool wide = cp.fuse_out < 0 && egress_wide(egress_args(out, cp));
        const bool iwide = cp.fuse_in < 0 && ingest_wide(ingest_args(in, cp));
        if (is_egress_wide_kernel(lru->second.egress_params.func) != wide ||
            is_ingest_wide_kernel(lru->second.ingest_params.func) != iwide) {
          cudaGraphExecDestroy(lru->second.exec);
          cudaGraphDestroy(lru->second.graph);
          cp.graphs.erase(lru);
        }
      }
      if (cp.graphs.size() >= static_cast<size_t>(graphs_per_plan())) {
        auto lru = cp.graphs.begin();
        for (auto jt = cp.graphs.begin(); jt != cp.graphs.end(); ++jt)
          if (jt->second.last_use < lru->second.last_use) lru = jt;
        g = lru->second;
        cp.graphs.erase(lru);
        g.ia = ingest_args(in, cp);
        g.ea = egress_args(out, cp);
        void* a1[] = {&g.ia, nullptr};
        if (cp.fuse_in >= 0) {  // the fused PQMF analysis carries the input pointer
          g.pin = pqmf_io_params(cp.fuse_in, cp, in, out);
          a1[0] = &g.pin;
          a1[1] = const_cast<float*>(plan->dops[cp.fuse_in].pq_k.data());
        }
        cudaKernelNodeParams kp = g.ingest_params;
        kp.kernelParams = a1;
        kp.extra = nullptr;
        ck(cudaGraphExecKernelNodeSetParams(g.exec, g.ingest_node, &kp), "ExecKernelNodeSetParams");
        void* a2[] = {&g.ea, nullptr};
        if (cp.fuse_out >= 0) {  // the fused PQMF synthesis carries the output pointer
          g.pout = pqmf_io_params(cp.fuse_out, cp, in, out);
          a2[0] = &g.pout;
          a2[1] = const_cast<float*>(plan->dops[cp.fuse_out].pq_k.data());
        }
        kp = g.egress_params;
        kp.kernelParams = a2;
        kp.extra = nullptr;
        ck(cudaGraphExecKernelNodeSetParams(g.exec, g.egress_node, &kp), "ExecKernelNodeSetParams");
      } else {
        ck(cudaStreamBeginCapture(capture_stream, cudaStreamCaptureModeThreadLocal), "BeginCapture");
        capturing = true;
        enqueue(in, out, cp, capture_stream, nullptr);
        capturing = false;
        cudaError_t le = cudaGetLastError();
        cudaGraph_t graph = nullptr;
        cudaError_t ee = cudaStreamEndCapture(capture_stream, &graph);
        ck(le, "launch (capture)");
        ck(ee, "EndCapture");
        g.graph = graph;
        size_t n = 0;
        ck(cudaGraphGetNodes(graph, nullptr, &n), "GraphGetNodes");
        std::vector<cudaGraphNode_t> nodes(n);
        ck(cudaGraphGetNodes(graph, nodes.data(), &n), "GraphGetNodes");
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType ty;
          ck(cudaGraphNodeGetType(nd, &ty), "NodeGetType");
          if (ty != cudaGraphNodeTypeKernel) continue;
          cudaKernelNodeParams kp;
          ck(cudaGraphKernelNodeGetParams(nd, &kp), "KernelNodeGetParams");
          const void* fin = cp.fuse_in >= 0 ? pqmf_kernel_ptr(1, 0, 0) : nullptr;
          const void* fout = nullptr;
          if (cp.fuse_out >= 0) {
            const ConvOp& so = plan->prog.ops[cp.fuse_out];
            fout = pqmf_kernel_ptr(2, so.pq_period, so.pq_mirror);
          }
          if (cp.fuse_in >= 0 ? kp.func == fin : (kp.func == ingest_kernel_ptr() || is_ingest_wide_kernel(kp.func))) {
            g.ingest_node = nd;
            g.ingest_params = kp;
          } else if (cp.fuse_out >= 0 ? kp.func == fout
                                      : (kp.func == egress_kernel_ptr() || is_egress_wide_kernel(kp.func))) {
            g.egress_node = nd;
            g.egress_params = kp;
          }
        }
        if (!g.ingest_node || !g.egress_node) fail(SC_ERR_INVALID_ARGUMENT, "graph I/O nodes not found");
        ck(cudaGraphInstantiate(&g.exec, graph, 0), "GraphInstantiate");
        ck(cudaGraphUpload(g.exec, s), "GraphUpload");
        g.ia = ingest_args(in, cp);
        g.ea = egress_args(out, cp);
      }
      it = cp.graphs.emplace(key, g).first;
    }
    it->second.last_use = ++use_clock;
    ck(cudaGraphLaunch(it->second.exec, s), "GraphLaunch");
    launched += cp.n_launch;
  }
  advance(F, cp);
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

// Host-buffer call: the step's input is copied H2D on its own stream, processed on the
// state's compute stream and copied back D2H on a third stream, with two device slots so
// call k+1's H2D and call k-1's D2H overlap call k's compute.  The H2D is ordered after the
// work already on `s` (entry event); host_wait(s) orders `s` after the last call's D2H.
void State::process_host(const float* h_in, float* h_out, int64_t F, cudaStream_t s) {
  process_host_io(h_in, h_out, F, s, false);
}

void State::process_host_bf16(const uint16_t* h_in, uint16_t* h_out, int64_t F, cudaStream_t s) {
  process_host_io(h_in, h_out, F, s, true);
}

// bf16 = true: the host buffers hold bf16 ([stream][C][T] like the fp32 ones) — half the PCIe
// bytes; the device widens the input to fp32 before the call and rounds the output (RN) after.
void State::process_host_io(const void* h_in, void* h_out, int64_t F, cudaStream_t s, bool bf16) {
  check_frames(F);
  if (!h_in || !h_out) fail(SC_ERR_INVALID_ARGUMENT, "null host pointer");
  const Program& pg = plan->prog;
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  const int64_t in_f = static_cast<int64_t>(streams) * pg.in_C * max_frames;
  const int64_t out_f = static_cast<int64_t>(streams) * pg.sink_C * (max_frames * pg.sink_rate.num / pg.sink_rate.den);
  if (!s_comp) {
    ck(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int k = 0; k < 2; ++k) {
      ck(cudaMalloc(&io_in[k], sizeof(float) * in_f), "cudaMalloc(io)");
      ck(cudaMalloc(&io_out[k], sizeof(float) * std::max<int64_t>(out_f, 1)), "cudaMalloc(io)");
      ck(cudaEventCreateWithFlags(&ev_entry[k], cudaEventDisableTiming), "EventCreate");
      ck(cudaEventCreateWithFlags(&ev_h2d[k], cudaEventDisableTiming), "EventCreate");
      ck(cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming), "EventCreate");
      ck(cudaEventCreateWithFlags(&ev_d2h[k], cudaEventDisableTiming), "EventCreate");
    }
    io_in_floats = in_f;
    io_out_floats = out_f;
  }
  if (bf16 && !io_in16[0]) {
    for (int k = 0; k < 2; ++k) {
      ck(cudaMalloc(&io_in16[k], sizeof(uint16_t) * in_f), "cudaMalloc(io bf16)");
      ck(cudaMalloc(&io_out16[k], sizeof(uint16_t) * std::max<int64_t>(out_f, 1)), "cudaMalloc(io bf16)");
    }
  }
  const int k = static_cast<int>(host_calls & 1);
  const size_t es = bf16 ? sizeof(uint16_t) : sizeof(float);
  const int64_t n_in = static_cast<int64_t>(streams) * pg.in_C * F;
  const int64_t n_out = static_cast<int64_t>(streams) * pg.sink_C * (F * pg.sink_rate.num / pg.sink_rate.den);
  const size_t in_bytes = es * static_cast<size_t>(n_in);
  const size_t out_bytes = es * static_cast<size_t>(n_out);
  ck(cudaEventRecord(ev_entry[k], s), "EventRecord");
  ck(cudaStreamWaitEvent(s_h2d, ev_entry[k], 0), "StreamWaitEvent");
  if (host_calls >= 2) ck(cudaStreamWaitEvent(s_h2d, ev_comp[k], 0), "StreamWaitEvent");  // slot k read
  ck(cudaMemcpyAsync(bf16 ? static_cast<void*>(io_in16[k]) : static_cast<void*>(io_in[k]), h_in, in_bytes,
                     cudaMemcpyHostToDevice, s_h2d), "H2D");
  ck(cudaEventRecord(ev_h2d[k], s_h2d), "EventRecord");
  ck(cudaStreamWaitEvent(s_comp, ev_h2d[k], 0), "StreamWaitEvent");
  if (host_calls >= 2) ck(cudaStreamWaitEvent(s_comp, ev_d2h[k], 0), "StreamWaitEvent");  // slot k drained
  if (bf16) launch_cast(io_in16[k], io_in[k], n_in, true, s_comp);  // bf16 -> fp32
  ck(cudaSetDevice(prev), "cudaSetDevice");
  process(io_in[k], io_out[k], F, s_comp);
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  if (bf16) launch_cast(io_out16[k], io_out[k], n_out, false, s_comp);  // fp32 -> bf16 (RN)
  ck(cudaEventRecord(ev_comp[k], s_comp), "EventRecord");
  ck(cudaStreamWaitEvent(s_d2h, ev_comp[k], 0), "StreamWaitEvent");
  ck(cudaMemcpyAsync(h_out, bf16 ? static_cast<void*>(io_out16[k]) : static_cast<void*>(io_out[k]), out_bytes,
                     cudaMemcpyDeviceToHost, s_d2h), "D2H");
  ck(cudaEventRecord(ev_d2h[k], s_d2h), "EventRecord");
  ++host_calls;
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

void State::host_wait(cudaStream_t s) {
  if (host_calls == 0) return;
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  ck(cudaStreamWaitEvent(s, ev_d2h[(host_calls - 1) & 1], 0), "StreamWaitEvent");
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

// Sink lag for a constant buffer length F from the current position: the largest shortfall
// E_k - N_sink_k over one period of calls (0 when F is a multiple of the ratio).
int64_t State::lag_for(int64_t F) const {
  const Program& pg = plan->prog;
  const int64_t Fs = F * pg.sink_rate.num / pg.sink_rate.den;
  int64_t P = pg.ratio / std::__gcd(F, pg.ratio);
  State* self = const_cast<State*>(this);
  const std::vector<int64_t> saveN = N;
  int64_t e = E, lag = 0;
  for (int64_t k = 0; k < P; ++k) {
    self->N = next_counts(F);
    e += Fs;
    lag = std::max(lag, e - N[pg.sink_buf]);
  }
  self->N = saveN;
  return lag;
}

void State::advance(int64_t F, const CallPlan& cp) {
  if (D < 0) D = lag_for(F);
  N = next_counts(F);
  for (size_t b = 0; b < pos.size(); ++b) pos[b] = cp.pos[b] + cp.T[b];
  E += cp.egress_T;
}

constexpr unsigned char kRedzoneByte = 0xA5;

void State::redzone_fill(cudaStream_t s) {
  for (size_t i = 0; i < buf_base.size(); ++i) {
    ck(cudaMemsetAsync(buf_base[i] - rz_gap, kRedzoneByte, rz_gap * 4, s), "redzone gap");
    ck(cudaMemset2DAsync(buf_base[i] + rz_used[i], buf_sstride[i] * 4, kRedzoneByte,
                         (buf_sstride[i] - rz_used[i]) * 4, streams, s), "redzone stream");
  }
  ck(cudaMemsetAsync(mem + mem_bytes / 4 - rz_gap, kRedzoneByte, rz_gap * 4, s), "redzone tail");
}

// guard bytes that no longer hold the fill pattern (-1: red zones disabled); synchronous
int64_t State::redzone_check() {
  if (rz_stream == 0) return -1;
  DeviceScope g(plan->device);
  ck(cudaDeviceSynchronize(), "redzone check");
  int64_t bad = 0;
  auto count = [&](const std::vector<unsigned char>& v) {
    for (unsigned char c : v) bad += c != kRedzoneByte;
  };
  std::vector<unsigned char> h;
  for (size_t i = 0; i < buf_base.size(); ++i) {
    h.assign(rz_gap * 4, 0);
    ck(cudaMemcpy(h.data(), buf_base[i] - rz_gap, h.size(), cudaMemcpyDeviceToHost), "redzone read");
    count(h);
    const int64_t w = (buf_sstride[i] - rz_used[i]) * 4;
    h.assign(w * streams, 0);
    ck(cudaMemcpy2D(h.data(), w, buf_base[i] + rz_used[i], buf_sstride[i] * 4, w, streams,
                    cudaMemcpyDeviceToHost), "redzone read");
    count(h);
  }
  h.assign(rz_gap * 4, 0);
  ck(cudaMemcpy(h.data(), mem + mem_bytes / 4 - rz_gap, h.size(), cudaMemcpyDeviceToHost), "redzone read");
  count(h);
  return bad;
}

void State::reset(const int* ids, int n_ids, cudaStream_t s) {
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  if (!ids) {
    ck(cudaMemsetAsync(mem, 0, mem_bytes, s), "cudaMemsetAsync");
    if (rz_stream > 0) redzone_fill(s);
    std::fill(N.begin(), N.end(), 0);
    std::fill(pos.begin(), pos.end(), 0);
    E = 0;
    D = -1;
  } else {
    if (n_ids < 0 || n_ids > streams) fail(SC_ERR_INVALID_ARGUMENT, "bad id count");
    for (int i = 0; i < n_ids; ++i)
      if (ids[i] < 0 || ids[i] >= streams) fail(SC_ERR_INVALID_ARGUMENT, "stream id out of range");
    // Phase state (buffers shorter than the compression ratio): every stream shares one
    // position, so strided layers window the new input at the shared phase.  Mid-period, a
    // reset stream would see windows misaligned for a fresh stream (SPEC reset = fresh init,
    // SPEC.md:281-284); at a period boundary nothing is pending anywhere and zeroing its
    // caches (the sink FIFO rows included) IS a fresh start.  So a subset reset is accepted
    // only at a boundary (a full reset, ids == NULL, is always exact).
    if (n_ids > 0 && phase_mode && N[0] % plan->prog.ratio != 0)
      fail(SC_ERR_INVALID_ARGUMENT,
           "subset reset in phase state only at a compression-period boundary (input frames so far " +
               std::to_string(N[0]) + " not a multiple of the ratio " + std::to_string(plan->prog.ratio) +
               "); reset all streams or reset after the period completes");
    if (n_ids > 0) {
      ck(cudaMemcpyAsync(d_ids, ids, sizeof(int) * n_ids, cudaMemcpyHostToDevice, s), "copy ids");
      // the caches currently start at each buffer's strip position
      std::vector<BufDesc> desc(reset_desc);
      for (BufDesc& d : desc) {
        const size_t b = static_cast<size_t>(std::find(buf_base.begin(), buf_base.end(), d.base) - buf_base.begin());
        d.base += pos[b] * d.C;
      }
      if (!desc.empty())
        ck(cudaMemcpyAsync(d_desc, desc.data(), desc.size() * sizeof(BufDesc), cudaMemcpyHostToDevice, s),
           "copy reset table");
      launch_reset_streams(d_desc, n_desc, d_ids, n_ids, reset_items, s);
      ck(cudaGetLastError(), "reset launch");
      // the host id array may be reused by the caller after return
      ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
  }
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

void conv1d_batched(const float* x, int batch, int M, int64_t L, const float* w, const float* b,
                    int N, int K, int S, int d, float* y, cudaStream_t s) {
  // check_conv_args (kernels.cpp:17-29)
  if (batch < 1 || M < 1 || N < 1 || K < 1 || L < 0) fail(SC_ERR_INVALID_ARGUMENT, "conv1d shape");
  if (S < 1 || d < 1) fail(SC_ERR_INVALID_ARGUMENT, "conv1d stride/dilation must be >= 1");
  const int64_t span = static_cast<int64_t>(K - 1) * d + 1;
  if (span > L)
    fail(SC_ERR_INPUT_TOO_SHORT, "conv1d input length " + std::to_string(L) +
                                     " shorter than kernel span " + std::to_string(span));
  if (!x || !w || !b || !y) fail(SC_ERR_INVALID_ARGUMENT, "null pointer");
  const int64_t Lo = (L - span) / S + 1;
  float *xt = nullptr, *wt = nullptr, *yt = nullptr;
  ck(cudaMallocAsync(&xt, sizeof(float) * batch * L * M, s), "cudaMallocAsync");
  ck(cudaMallocAsync(&wt, sizeof(float) * static_cast<int64_t>(K) * M * N, s), "cudaMallocAsync");
  ck(cudaMallocAsync(&yt, sizeof(float) * batch * Lo * N, s), "cudaMallocAsync");
  IngestArgs ia{x, xt, L * M, M, static_cast<int>(L), 0, batch};
  launch_ingest(ia, s);
  launch_relayout_w(w, N, M, K, wt, s);
  ConvParams p{};
  p.in = xt;
  p.in_sstride = L * M;
  p.in_fstride = M;
  p.cin = M;
  p.row_step = S;
  p.tap_step = d;
  p.taps = K;
  p.w = wt;
  p.bias = b;
  p.nout = N;
  p.out = yt;
  p.out_sstride = Lo * N;
  p.out_rstride = N;
  p.t_out = static_cast<int>(Lo);
  p.streams = batch;
  launch_conv_simt(p, s);
  EgressArgs ea{};
  ea.buf = yt;
  ea.sstride = Lo * N;
  ea.fstride = N;
  ea.C = N;
  ea.T = static_cast<int>(Lo);
  ea.streams = batch;
  ea.out = y;
  launch_egress(ea, s);
  ck(cudaGetLastError(), "conv1d launch");
  cudaFreeAsync(xt, s);
  cudaFreeAsync(wt, s);
  cudaFreeAsync(yt, s);
}

}  // namespace scb
