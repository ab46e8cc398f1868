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

#include <algorithm>
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
                      uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2, bool bf16 = false) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(SC_ERR_CUDA_BASE, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

bool tc_disabled() {
  const char* e = std::getenv("SC_DISABLE_TC");
  return e && std::atoi(e) != 0;
}

// Decide whether an op runs on the tensor-core kernel and build its hi/lo weight planes.
void plan_tc(const Program& pg, size_t i, int precision, DevOp& d, std::vector<float>& wtc) {
  const ConvOp& op = pg.ops[i];
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
    // the output tile (BN/2 columns) must be a whole 32-column TMA box
    if (op.nout > 64 && op.nout % 64 != 0) return;
    d.BN = (op.nout % 128 == 0) ? 128 : 64;
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
  // fp32: [2 (hi, lo)][N][Kpad] floats; bf16: [N][Kpad] bf16 (round-to-nearest) packed in floats
  wtc.assign(d.bf16 ? static_cast<size_t>((N * Kpad + 1) / 2) : static_cast<size_t>(2 * N * Kpad), 0.f);
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
        } else {
          const float hi = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, w) & 0xFFFFE000u);
          wtc[o] = hi;
          wtc[static_cast<size_t>(N * Kpad) + o] = w - hi;
        }
      }
}
}  // namespace

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
  auto plan = std::make_unique<Plan>();
  plan->prog = lower_graph(nodes, n_nodes, W, nW, in_C);
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
  int64_t total = 0;
  std::vector<int64_t> woff, boff, toff;
  for (size_t i = 0; i < nops; ++i) {
    const ConvOp& op = plan->prog.ops[i];
    woff.push_back(total);
    total += round_up(static_cast<int64_t>(op.w.size()), 64);
    boff.push_back(total);
    total += round_up(static_cast<int64_t>(op.bias.size()), 64);
    toff.push_back(total);
    total += round_up(static_cast<int64_t>(wtc[i].size()), 64);
  }
  std::vector<float> host(static_cast<size_t>(std::max<int64_t>(total, 1)), 0.f);
  for (size_t i = 0; i < nops; ++i) {
    const ConvOp& op = plan->prog.ops[i];
    std::memcpy(host.data() + woff[i], op.w.data(), op.w.size() * sizeof(float));
    std::memcpy(host.data() + boff[i], op.bias.data(), op.bias.size() * sizeof(float));
    if (!wtc[i].empty()) std::memcpy(host.data() + toff[i], wtc[i].data(), wtc[i].size() * sizeof(float));
  }
  ck(cudaMalloc(&plan->wmem, host.size() * sizeof(float)), "cudaMalloc(weights)");
  ck(cudaMemcpy(plan->wmem, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice),
     "cudaMemcpy(weights)");
  for (size_t i = 0; i < nops; ++i) {
    DevOp& d = plan->dops[i];
    d.w = plan->wmem + woff[i];
    d.bias = plan->wmem + boff[i];
    if (d.kernel == KERNEL_TC) {
      const ConvOp& op = plan->prog.ops[i];
      d.wtc = plan->wmem + toff[i];
      const uint64_t Kpad = static_cast<uint64_t>(d.taps_view) * d.cin_view_pad;
      if (d.bf16)
        d.map_w = make_map3(d.wtc, Kpad, op.nout, 1, Kpad * 2, static_cast<uint64_t>(op.nout) * Kpad * 2, 32,
                            d.BN, 1, true);
      else
        d.map_w = make_map3(d.wtc, Kpad, op.nout, 2, Kpad * 4, static_cast<uint64_t>(op.nout) * Kpad * 4, 32,
                            d.BN, 1);
    }
  }
  plan->desc = plan->prog.describe();
  ck(cudaSetDevice(prev), "cudaSetDevice");
  return plan;
}

// --------------------------------------------------------------------------- state
State::~State() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  for (auto& kv : graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  if (capture_stream) cudaStreamDestroy(capture_stream);
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
  if (max_frames % pg.ratio != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO,
         "max_frames " + std::to_string(max_frames) + " not a multiple of ratio " + std::to_string(pg.ratio));
  auto st = std::make_unique<State>();
  st->plan = plan;
  st->streams = streams;
  st->max_frames = max_frames;
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  int64_t total = 0;
  std::vector<int64_t> off;
  for (const BufferSpec& b : pg.bufs) {
    const int64_t T = max_frames * b.rate.num / b.rate.den;
    const int64_t sstride = round_up((b.cache + T) * b.C, 32);
    st->buf_sstride.push_back(sstride);
    off.push_back(total);
    total += round_up(sstride * streams, 64);
    st->cache_bytes_per_stream += b.cache * b.C * 4;
  }
  st->mem_bytes = total * 4;
  ck(cudaMalloc(&st->mem, std::max<int64_t>(st->mem_bytes, 256)), "cudaMalloc(state)");
  ck(cudaMemset(st->mem, 0, std::max<int64_t>(st->mem_bytes, 256)), "cudaMemset(state)");
  for (size_t i = 0; i < pg.bufs.size(); ++i) st->buf_base.push_back(st->mem + off[i]);
  // carry / reset table: buffers with a cache
  std::vector<BufDesc> desc;
  int64_t items = 0, ritems = 0;
  for (size_t i = 0; i < pg.bufs.size(); ++i) {
    const BufferSpec& b = pg.bufs[i];
    if (b.cache == 0) continue;
    BufDesc d{};
    d.base = st->buf_base[i];
    d.sstride = st->buf_sstride[i];
    d.item0 = items;
    d.ritem0 = ritems;
    d.C = b.C;
    d.cache = static_cast<int>(b.cache);
    d.rnum = static_cast<int>(b.rate.num);
    d.rden = static_cast<int>(b.rate.den);
    items += static_cast<int64_t>(streams) * b.C;
    ritems += b.C;
    desc.push_back(d);
  }
  if (desc.size() > 64) fail(SC_ERR_UNSUPPORTED_FORMAT, "more than 64 cached buffers");
  st->n_desc = static_cast<int>(desc.size());
  st->carry_items = items;
  st->reset_items = ritems;
  if (!desc.empty()) {
    ck(cudaMalloc(&st->d_desc, desc.size() * sizeof(BufDesc)), "cudaMalloc(desc)");
    ck(cudaMemcpy(st->d_desc, desc.data(), desc.size() * sizeof(BufDesc), cudaMemcpyHostToDevice),
       "cudaMemcpy(desc)");
  }
  ck(cudaMalloc(&st->d_ids, sizeof(int) * streams), "cudaMalloc(ids)");
  ck(cudaStreamCreateWithFlags(&st->capture_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaSetDevice(prev), "cudaSetDevice");
  return st;
}

ConvParams State::conv_params(size_t i, int64_t F) const {
  const Program& pg = plan->prog;
  const ConvOp& op = pg.ops[i];
  const BufferSpec& bi = pg.bufs[op.in_buf];
  const BufferSpec& bo = pg.bufs[op.out_buf];
  const int64_t Tin = F * op.in_rate.num / op.in_rate.den;
  ConvParams p{};
  p.in = buf_base[op.in_buf];
  p.in_sstride = buf_sstride[op.in_buf];
  p.in_fstride = bi.C;
  p.in_off = op.in_off;
  p.cin = op.cin;
  p.in_f0 = static_cast<int>(bi.cache - op.look);
  p.row_step = op.row_step;
  p.tap_step = op.tap_step;
  p.taps = op.taps;
  p.w = plan->dops[i].w;
  p.bias = plan->dops[i].bias;
  p.nout = op.nout;
  p.out = buf_base[op.out_buf];
  p.out_sstride = buf_sstride[op.out_buf];
  p.out_base = bo.cache * bo.C;
  p.out_rstride = op.out_rstride;
  p.t_out = static_cast<int>(op.convt ? Tin : Tin / op.S);
  p.streams = streams;
  p.pre_act = op.pre_act;
  p.pre_alpha = op.pre_alpha;
  p.post_act = op.post_act;
  p.post_alpha = op.post_alpha;
  p.gate = op.gate ? 1 : 0;
  if (op.res_buf >= 0) {
    const BufferSpec& br = pg.bufs[op.res_buf];
    p.res = buf_base[op.res_buf];
    p.res_sstride = buf_sstride[op.res_buf];
    p.res_fstride = br.C;
    p.res_off = op.res_off;
    p.res_f0 = static_cast<int>(br.cache - op.res_delay);
    p.res_act = op.res_act;
    p.res_alpha = op.res_alpha;
  }
  return p;
}

IngestArgs State::ingest_args(const float* in, int64_t F) const {
  const Program& pg = plan->prog;
  IngestArgs a{};
  a.in = in;
  a.buf = buf_base[0];
  a.sstride = buf_sstride[0];
  a.C = pg.in_C;
  a.T = static_cast<int>(F);
  a.cache = static_cast<int>(pg.bufs[0].cache);
  a.streams = streams;
  return a;
}

EgressArgs State::egress_args(float* out, int64_t F) const {
  const Program& pg = plan->prog;
  const BufferSpec& b = pg.bufs[pg.sink_buf];
  EgressArgs a{};
  a.buf = buf_base[pg.sink_buf];
  a.sstride = buf_sstride[pg.sink_buf];
  a.fstride = b.C;
  a.off = pg.sink_off;
  a.C = pg.sink_C;
  a.T = static_cast<int>(F * pg.sink_rate.num / pg.sink_rate.den);
  a.cache = static_cast<int>(b.cache);
  a.streams = streams;
  a.act = pg.sink_act;
  a.alpha = pg.sink_alpha;
  a.out = out;
  return a;
}

int State::launches(int64_t F) const {
  (void)F;
  return 2 + static_cast<int>(plan->prog.ops.size()) + (n_desc > 0 ? 1 : 0);
}

std::string State::launch_name(int64_t F, int i) const {
  const int nops = static_cast<int>(plan->prog.ops.size());
  if (i == 0) return "ingest";
  if (i >= 1 && i <= nops) {
    const ConvOp& op = plan->prog.ops[i - 1];
    return "op" + std::to_string(i - 1) + " " + op.name + " [" +
           (plan->dops[i - 1].kernel == KERNEL_TC ? (plan->dops[i - 1].bf16 ? "tc-bf16" : "tc") : "simt") + "]";
  }
  if (i == nops + 1) return "egress";
  if (i == nops + 2 && n_desc > 0) return "carry";
  (void)F;
  return "";
}

const std::vector<TcLaunch>& State::tc_for(int64_t F) {
  auto it = tc_launches.find(F);
  if (it != tc_launches.end()) return it->second;
  const Program& pg = plan->prog;
  std::vector<TcLaunch> v(pg.ops.size());
  for (size_t i = 0; i < pg.ops.size(); ++i) {
    const DevOp& d = plan->dops[i];
    if (d.kernel != KERNEL_TC) continue;
    const ConvOp& op = pg.ops[i];
    const BufferSpec& bi = pg.bufs[op.in_buf];
    const ConvParams cp = conv_params(i, F);
    const int64_t Tmax_in = max_frames * bi.rate.num / bi.rate.den;
    const int S = d.view_S;
    const uint64_t bufC_view = static_cast<uint64_t>(bi.C) * S;
    const uint64_t rows_view = static_cast<uint64_t>((bi.cache + Tmax_in) / S);
    TcParams& p = v[i].p;
    p.BN = d.BN;
    p.bf16 = d.bf16 ? 1 : 0;
    const int t_out = cp.t_out;
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
    p.cblocks = d.cin_view_pad / 32;
    p.n_kblocks = d.taps_view * p.cblocks;
    p.a_c0 = S > 1 ? 0 : op.in_off;
    p.a_row0 = static_cast<int>((bi.cache - op.look) / S);
    p.a_tap_rows = d.tap_rows;
    p.pre_act = cp.pre_act;
    p.pre_alpha = cp.pre_alpha;
    p.post_act = cp.post_act;
    p.post_alpha = cp.post_alpha;
    p.gate = cp.gate;
    p.nout = cp.nout;
    p.t_out = t_out;
    p.streams = streams;
    p.bias = cp.bias;
    p.out = cp.out;
    p.out_sstride = cp.out_sstride;
    p.out_base = cp.out_base;
    p.out_rstride = cp.out_rstride;
    p.res = cp.res;
    p.res_sstride = cp.res_sstride;
    p.res_fstride = cp.res_fstride;
    p.res_off = cp.res_off;
    p.res_f0 = cp.res_f0;
    p.res_act = cp.res_act;
    p.res_alpha = cp.res_alpha;
    {
      const char* dbg = std::getenv("SC_TC_DEBUG");
      p.debug = dbg ? std::atoi(dbg) : 0;
      const char* tr = std::getenv("SC_TC_TRACE_OP");
      if (tr && std::atoi(tr) == static_cast<int>(i)) p.debug |= 32;
    }
    v[i].map_a = make_map3(buf_base[op.in_buf], bufC_view, rows_view, streams, bufC_view * 4,
                           static_cast<uint64_t>(buf_sstride[op.in_buf]) * 4, 32,
                           static_cast<uint32_t>(p.R), static_cast<uint32_t>(p.G));
    // output rows start at out_base; rows >= t_out and streams >= n_streams are clipped by TMA
    v[i].map_out = make_map3(cp.out + cp.out_base, static_cast<uint64_t>(cp.out_rstride),
                             static_cast<uint64_t>(t_out), streams, static_cast<uint64_t>(cp.out_rstride) * 4,
                             static_cast<uint64_t>(cp.out_sstride) * 4, 32, static_cast<uint32_t>(p.R),
                             static_cast<uint32_t>(p.G));
    if (cp.res) {
      v[i].map_res = make_map3(cp.res + static_cast<int64_t>(cp.res_f0) * cp.res_fstride,
                               static_cast<uint64_t>(cp.res_fstride), static_cast<uint64_t>(t_out), streams,
                               static_cast<uint64_t>(cp.res_fstride) * 4,
                               static_cast<uint64_t>(cp.res_sstride) * 4, 32, static_cast<uint32_t>(p.R),
                               static_cast<uint32_t>(p.G));
    } else {
      v[i].map_res = v[i].map_out;  // unused
    }
  }
  return tc_launches.emplace(F, std::move(v)).first->second;
}

void State::enqueue(const float* in, float* out, int64_t F, cudaStream_t s, cudaEvent_t* ev) {
  int e = 0;
  const std::vector<TcLaunch>& tcl = tc_for(F);
  if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  launch_ingest(ingest_args(in, F), s);
  if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  for (size_t i = 0; i < plan->prog.ops.size(); ++i) {
    if (plan->dops[i].kernel == KERNEL_TC) {
      launch_conv_tc(tcl[i].map_a, plan->dops[i].map_w, tcl[i].map_out, tcl[i].map_res, tcl[i].p, s);
    } else {
      launch_conv_simt(conv_params(i, F), s);
    }
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
  launch_egress(egress_args(out, F), s);
  if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  if (n_desc > 0) {
    launch_carry(d_desc, n_desc, streams, carry_items, F, s);
    if (ev) ck(cudaEventRecord(ev[e++], s), "EventRecord");
  }
}

void State::profile(const float* in, float* out, int64_t F, int steps, float* ms, cudaStream_t s) {
  check_frames(F);
  if (steps < 1) fail(SC_ERR_INVALID_ARGUMENT, "steps must be >= 1");
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  const int n = launches(F);
  std::vector<cudaEvent_t> ev(static_cast<size_t>(n + 1) * steps);
  for (auto& e : ev) ck(cudaEventCreate(&e), "EventCreate");
  for (int k = 0; k < steps; ++k) enqueue(in, out, F, s, ev.data() + static_cast<size_t>(k) * (n + 1));
  ck(cudaGetLastError(), "launch");
  ck(cudaStreamSynchronize(s), "StreamSynchronize");
  for (int i = 0; i < n; ++i) ms[i] = 0.f;
  for (int k = 0; k < steps; ++k)
    for (int i = 0; i < n; ++i) {
      float t = 0.f;
      ck(cudaEventElapsedTime(&t, ev[static_cast<size_t>(k) * (n + 1) + i],
                              ev[static_cast<size_t>(k) * (n + 1) + i + 1]),
         "EventElapsedTime");
      ms[i] += t / steps;
    }
  for (auto& e : ev) cudaEventDestroy(e);
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

void State::check_frames(int64_t F) const {
  if (F <= 0) fail(SC_ERR_INVALID_ARGUMENT, "frames must be positive");
  if (F % plan->prog.ratio != 0)
    fail(SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO, "buffer length " + std::to_string(F) +
                                                  " is not a multiple of the compression ratio " +
                                                  std::to_string(plan->prog.ratio));
  if (F > max_frames)
    fail(SC_ERR_INVALID_ARGUMENT, "buffer length " + std::to_string(F) + " exceeds max_frames " +
                                      std::to_string(max_frames));
}

void State::process(const float* in, float* out, int64_t F, cudaStream_t s) {
  check_frames(F);
  if (!in || !out) fail(SC_ERR_INVALID_ARGUMENT, "null I/O pointer");
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  if (!use_graphs) {
    enqueue(in, out, F, s, nullptr);
    ck(cudaGetLastError(), "launch");
    ck(cudaSetDevice(prev), "cudaSetDevice");
    return;
  }
  const auto key = std::make_tuple(F, in, out);
  auto it = graphs.find(key);
  if (it == graphs.end()) {
    // reuse the least recently used graph of this length once 8 pointer pairs exist
    int same = 0;
    auto lru = graphs.end();
    for (auto jt = graphs.begin(); jt != graphs.end(); ++jt) {
      if (std::get<0>(jt->first) != F) continue;
      ++same;
      if (lru == graphs.end() || jt->second.last_use < lru->second.last_use) lru = jt;
    }
    GraphEntry g;
    if (same >= 8) {
      g = lru->second;
      graphs.erase(lru);
      g.ia = ingest_args(in, F);
      g.ea = egress_args(out, F);
      void* a1[] = {&g.ia};
      cudaKernelNodeParams kp = g.ingest_params;
      kp.kernelParams = a1;
      kp.extra = nullptr;
      ck(cudaGraphExecKernelNodeSetParams(g.exec, g.ingest_node, &kp), "ExecKernelNodeSetParams");
      void* a2[] = {&g.ea};
      kp = g.egress_params;
      kp.kernelParams = a2;
      kp.extra = nullptr;
      ck(cudaGraphExecKernelNodeSetParams(g.exec, g.egress_node, &kp), "ExecKernelNodeSetParams");
    } else {
      ck(cudaStreamBeginCapture(capture_stream, cudaStreamCaptureModeThreadLocal), "BeginCapture");
      enqueue(in, out, F, capture_stream, nullptr);
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
        if (kp.func == ingest_kernel_ptr()) {
          g.ingest_node = nd;
          g.ingest_params = kp;
        } else if (kp.func == egress_kernel_ptr()) {
          g.egress_node = nd;
          g.egress_params = kp;
        }
      }
      if (!g.ingest_node || !g.egress_node) fail(SC_ERR_INVALID_ARGUMENT, "graph I/O nodes not found");
      ck(cudaGraphInstantiate(&g.exec, graph, 0), "GraphInstantiate");
      ck(cudaGraphUpload(g.exec, s), "GraphUpload");
      g.ia = ingest_args(in, F);
      g.ea = egress_args(out, F);
    }
    it = graphs.emplace(key, g).first;
  }
  GraphEntry& g = it->second;
  g.last_use = ++use_clock;
  ck(cudaGraphLaunch(g.exec, s), "GraphLaunch");
  ck(cudaSetDevice(prev), "cudaSetDevice");
}

void State::reset(const int* ids, int n_ids, cudaStream_t s) {
  int prev = 0;
  ck(cudaGetDevice(&prev), "cudaGetDevice");
  ck(cudaSetDevice(plan->device), "cudaSetDevice");
  if (!ids) {
    ck(cudaMemsetAsync(mem, 0, mem_bytes, s), "cudaMemsetAsync");
  } else {
    if (n_ids < 0 || n_ids > streams) fail(SC_ERR_INVALID_ARGUMENT, "bad id count");
    for (int i = 0; i < n_ids; ++i)
      if (ids[i] < 0 || ids[i] >= streams) fail(SC_ERR_INVALID_ARGUMENT, "stream id out of range");
    if (n_ids > 0) {
      ck(cudaMemcpyAsync(d_ids, ids, sizeof(int) * n_ids, cudaMemcpyHostToDevice, s), "copy ids");
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
