/*
 * streamconv_b200.h — C-ABI of the B200-native multi-stream cached-padding engine.
 *
 * This is the drop-in boundary for the hot path of arXiv 2204.07064 as specified by the
 * reference (`/root/reference/SPEC.md`, module `stream_runtime`) and implemented, for its
 * arithmetic core, by `proj/src/kernels.cpp`.  The reference is an in-process C++ API in
 * `namespace streamconv` with no C ABI; every entry point below names the
 * reference function it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - Every function returns an `int` status: SC_OK (0) or 1 + the ordinal of the reference
 *     `streamconv::ErrCode` (proj/include/streamconv/error.hpp:8-29), or SC_ERR_CUDA_BASE +
 *     cudaError_t.  `sc_last_error()` returns the message of the last failure on the calling
 *     thread, formatted like `streamconv::Error::what()` ("<ErrCode>: <msg>", error.hpp:59-60).
 *   - Signals at the boundary use the reference layout (SignalTensor, tensor.hpp:14-48):
 *     fp32, channel-major `[channels][length]` per stream; a batch of streams is
 *     `[stream][channels][length]` contiguous.  Device pointers unless stated otherwise.
 *   - Conv weights use the reference `Kernel` layout (tensor.hpp:52-88): weights `[n][m][k]`
 *     followed by bias `[n]`, fp32, in ONE host array addressed by `sc_node.weight_offset`.
 *   - `stream` arguments are `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 */
#ifndef STREAMCONV_B200_H
#define STREAMCONV_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SC_API __attribute__((visibility("default")))
#else
#define SC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + streamconv::ErrCode ordinal (error.hpp:8-29) ------------------- */
enum sc_status {
  SC_OK = 0,
  SC_ERR_INVALID_ARGUMENT = 1,            /* ErrCode::InvalidArgument */
  SC_ERR_INPUT_TOO_SHORT = 2,             /* ErrCode::InputTooShort */
  SC_ERR_CHANNEL_MISMATCH = 3,            /* ErrCode::ChannelMismatch */
  SC_ERR_CYCLE_DETECTED = 4,              /* ErrCode::CycleDetected */
  SC_ERR_DANGLING_NODE = 5,               /* ErrCode::DanglingNode */
  SC_ERR_RATE_MISMATCH_AT_SUM = 6,        /* ErrCode::RateMismatchAtSum */
  SC_ERR_MALFORMED_GRAPH = 7,             /* ErrCode::MalformedGraph */
  SC_ERR_NOT_CAUSAL = 8,                  /* ErrCode::NotCausal */
  SC_ERR_PADDING_NOT_STREAMABLE = 9,      /* ErrCode::PaddingNotStreamable */
  SC_ERR_INTERNAL_NON_INTEGER_DELAY = 10, /* ErrCode::InternalNonIntegerDelay */
  SC_ERR_BUFFER_NOT_MULTIPLE_OF_RATIO = 11, /* ErrCode::BufferNotMultipleOfRatio */
  SC_ERR_LENGTH_NOT_MULTIPLE_OF_RATIO = 12, /* ErrCode::LengthNotMultipleOfRatio */
  SC_ERR_CHUNK_TOO_SMALL = 13,            /* ErrCode::ChunkTooSmall */
  SC_ERR_LENGTH_MISMATCH = 14,            /* ErrCode::LengthMismatch */
  SC_ERR_ZERO_ENERGY = 15,                /* ErrCode::ZeroEnergy */
  SC_ERR_VERSION_MISMATCH = 16,           /* ErrCode::VersionMismatch */
  SC_ERR_CORRUPT_BLOB = 17,               /* ErrCode::CorruptBlob */
  SC_ERR_SCHEMA_ERROR = 18,               /* ErrCode::SchemaError */
  SC_ERR_UNSUPPORTED_FORMAT = 19,         /* ErrCode::UnsupportedFormat */
  SC_ERR_MALFORMED_HEADER = 20,           /* ErrCode::MalformedHeader */
  SC_ERR_CUDA_BASE = 1000                 /* 1000 + cudaError_t */
};

/* ---- activation kinds: streamconv::Act (kernels.hpp:9) --------------------------------- */
enum sc_act { SC_ACT_IDENTITY = 0, SC_ACT_TANH = 1, SC_ACT_LEAKY_RELU = 2 };

/* ---- graph nodes ------------------------------------------------------------------------
 * A model is a flat, topologically ordered node list: a sequential stack with nested
 * residual scopes.  This is the subset of SPEC graph_ir that the
 * north-star models need: Conv / ZeroUpsample+Conv (ConvTranspose1d) /
 * Activation / Fanout+Sum with an identity skip / channel gate / slice.
 * Paddings are the ORIGINAL (possibly non-causal) ones; plan creation runs the causalize
 * rewrite and inserts the Eq. (2) and branch-alignment delays itself.  */
enum sc_node_kind {
  SC_NODE_CONV = 0,      /* conv1d(pad(x,(L,R)), k, stride, dilation)        kernels.cpp:73  */
  SC_NODE_CONVT = 1,     /* conv1d(pad(zero_upsample(x,stride),(L,R)), k)   kernels.cpp:106 */
  SC_NODE_ACT = 2,       /* activation(x, act, alpha)                        kernels.cpp:119 */
  SC_NODE_RES_BEGIN = 3, /* Fanout: start of a residual branch; skip = identity           */
  SC_NODE_RES_END = 4,   /* Sum(branch, Delay_A(skip)) with A from branch_alignment        */
  SC_NODE_GATE = 5,      /* y[c] = tanh(x[c]) * sigmoid(x[c + C/2]), C -> C/2  (RAVE head) */
  SC_NODE_SLICE = 6      /* keep channels [slice_begin, slice_begin + slice_count)         */
};

typedef struct sc_node {
  int32_t kind;          /* enum sc_node_kind */
  int32_t in_channels;   /* CONV/CONVT: M */
  int32_t out_channels;  /* CONV/CONVT: N */
  int32_t taps;          /* CONV/CONVT: K */
  int32_t stride;        /* CONV: S;  CONVT: upsampling factor */
  int32_t dilation;      /* CONV: d (CONVT: must be 1) */
  int64_t pad_left;      /* original PaddingSpec{left,right} (tensor.hpp:90-95) */
  int64_t pad_right;
  int32_t act;           /* ACT: enum sc_act */
  float alpha;           /* ACT: leaky_relu slope (reference default 0.01f, kernels.hpp:32) */
  int64_t weight_offset; /* CONV/CONVT: float offset of weights[N][M][K] then bias[N] */
  int32_t slice_begin;   /* SLICE */
  int32_t slice_count;   /* SLICE */
  int32_t hint;          /* enum sc_hint: structure the planner may exploit (verified) */
} sc_node;

/* Planner hints.  SC_HINT_PQMF marks a CONV / CONVT node whose weights are a cosine-modulated
 * filter bank (sc_pqmf_filters): the plan factors them into the polyphase + modulation form
 * (5x fewer MACs) after checking the factorisation reproduces every weight to 1e-6, and
 * otherwise runs the node as a generic conv.  Results are unaffected beyond fp32 rounding. */
enum sc_hint { SC_HINT_NONE = 0, SC_HINT_PQMF = 1 };

/* arithmetic variants of the dense path */
enum sc_precision {
  SC_PREC_FP32 = 0,      /* fp32-accurate: FFMA or 3xTF32 tensor-core, fp32 accumulate */
  SC_PREC_BF16 = 1       /* bf16 operands, fp32 accumulate (separately stated bound)     */
};

typedef struct sc_plan sc_plan;
typedef struct sc_state sc_state;

/* ---- library / errors ------------------------------------------------------------------ */
SC_API const char* sc_last_error(void);
SC_API const char* sc_version(void);
SC_API const char* sc_status_name(int status); /* streamconv::to_string(ErrCode) (error.hpp:31-55) */

/* ---- causalize arithmetic -------------------------------------------- */
/* Eq. (2): D_a = (S - ((R + D_c) mod S)) mod S */
SC_API int64_t sc_delay_for_stride(int64_t stride, int64_t right_pad, int64_t cumulated_delay);
/* A_i = max_j D_j - D_i */
SC_API int sc_branch_alignment(const int64_t* delays, int32_t n, int64_t* out);

/* ---- plans: a validated + causalized graph with device-resident weights ---------------- */
/* Replaces: SPEC causalize(g) + weight upload.  `weights_host` holds every
 * node's Kernel (tensor.hpp:52-88).  `device` is the CUDA ordinal; device = -1 creates a
 * host-only plan (validation, causalize, ledger and lowering only; no states, no GPU).     */
SC_API int sc_plan_create(const sc_node* nodes, int32_t n_nodes, const float* weights_host,
                   int64_t n_weights, int32_t in_channels, int32_t precision, int32_t device,
                   sc_plan** out);
SC_API int sc_plan_destroy(sc_plan* plan);
/* SPEC compression_ratio: granularity of the buffer length. */
SC_API int sc_plan_ratio(const sc_plan* plan, int64_t* ratio);
/* Sink rate ratio: output samples per input sample = num/den. */
SC_API int sc_plan_sink_rate(const sc_plan* plan, int64_t* num, int64_t* den, int32_t* out_channels);
/* SPEC latency_of: total input->output latency in input samples. */
SC_API int sc_plan_latency(const sc_plan* plan, int64_t* samples);
/* SPEC closed-form state size: sum over causalized Conv caches and Delay
 * rings of (len x channels x 4) bytes per stream.                                      */
SC_API int sc_plan_state_bytes(const sc_plan* plan, int64_t* bytes_per_stream);
/* Algorithmic work per stream per input sample (no zero-stuffed MACs, SPEC.md:405 fixed). */
SC_API int sc_plan_macs_per_sample(const sc_plan* plan, double* macs);
/* Number of fused conv ops, and op i's algorithmic MACs per stream per input sample. */
SC_API int sc_plan_num_ops(const sc_plan* plan, int32_t* n);
SC_API int sc_plan_op_macs(const sc_plan* plan, int32_t i, double* macs);
/* Human-readable lowering summary (buffers, ops, kernels), valid until plan destroy. */
SC_API const char* sc_plan_describe(const sc_plan* plan);

/* ---- stream states: SPEC StreamState for a batch of independent streams ----------------- */
/* Replaces: init_state, one per stream, zeroed.  `max_frames` = largest
 * per-call buffer length (input samples per stream) this state will be used with.          */
SC_API int sc_state_create(const sc_plan* plan, int32_t n_streams, int64_t max_frames, sc_state** out);
SC_API int sc_state_destroy(sc_state* state);
/* Replaces: reset for the listed streams (NULL ids = all). Async. */
SC_API int sc_state_reset(sc_state* state, const int32_t* stream_ids, int32_t n_ids, void* stream);
/* Device bytes actually held by the state: caches + step working buffers + the cached call
   plans (carry tables; at most 32 plans are kept, least recently used evicted first). */
SC_API int sc_state_device_bytes(const sc_state* state, int64_t* bytes);
/* Resident cache bytes per stream (<= sc_plan_state_bytes: skip delays share conv caches). */
SC_API int sc_state_cache_bytes(const sc_state* state, int64_t* bytes_per_stream);
/* Debug: with SC_REDZONE=1 in the environment at sc_state_create, every stream's strip and
 * every buffer is followed by guard bytes holding a fill pattern; this counts the guard bytes
 * that were overwritten since (out-of-bounds device writes).  *violations = -1 when the state
 * has no red zones.  Synchronous (waits for the device).  No reference counterpart: a memcheck
 * substitute (compute-sanitizer is unavailable on the GPU pool). */
SC_API int sc_state_redzone_check(sc_state* state, int64_t* violations);

/* Replaces: process_buffer for every stream of `state` at once.
 * d_in  : [n_streams][in_channels][frames]  fp32 device
 * d_out : [n_streams][out_channels][frames * sink_rate] fp32 device
 * frames must be a positive multiple of sc_plan_ratio and <= max_frames.  Asynchronous on
 * `stream`; the steady-state launch sequence is replayed from a cached CUDA graph.        */
SC_API int sc_process(sc_state* state, const float* d_in, float* d_out, int64_t frames, void* stream);
/* Same call with HOST buffers (the reference's process_buffer takes host SignalTensors):
 * h_in / h_out as above but in host memory — pinned (cudaHostAlloc/cudaHostRegister) for
 * asynchronous copies.  The H2D copy, the compute and the D2H copy run on three internal
 * streams with two device slots, so consecutive calls overlap each other's transfers.  The
 * H2D is ordered after the work already queued on `stream`; call sc_process_host_wait to
 * order `stream` after the last call's D2H (then synchronize it before reading h_out).  As
 * with cudaMemcpyAsync, h_in must not be overwritten before its copy has run.            */
SC_API int sc_process_host(sc_state* state, const float* h_in, float* h_out, int64_t frames,
                           void* stream);
SC_API int sc_process_host_wait(sc_state* state, void* stream);
/* sc_process_host with bf16 host buffers (uint16 bit patterns, same [stream][C][T] layouts):
 * half the PCIe bytes; the device widens the input to fp32 and rounds the fp32 output to bf16
 * (nearest-even) — for the bf16-operand variant, whose stated error bound covers it. */
SC_API int sc_process_host_bf16(sc_state* state, const uint16_t* h_in, uint16_t* h_out,
                                int64_t frames, void* stream);
/* Launch slots of one sc_process call (profile layout): carry (wrap-around calls only, see
 * DESIGN.md §3 strips), ingest, one per firing op, egress. */
SC_API int sc_process_launches(const sc_state* state, int64_t frames, int32_t* n);
/* Kernels launched so far by this state (eager, graph-replayed or profiled calls): the exact
 * launch count of a timed region is the difference of two readings. */
SC_API int sc_state_launch_total(const sc_state* state, int64_t* total);
/* Measurement: run `steps` calls WITHOUT graph replay with CUDA events between launches;
 * ms_per_launch[i] = mean device time of launch i (sc_process_launches entries).          */
SC_API int sc_state_profile(sc_state* state, const float* d_in, float* d_out, int64_t frames,
                            int32_t steps, float* ms_per_launch, void* stream);
/* Name of launch i of one call ("ingest", "op3 conv 128->128 K3 d9 [simt]", "carry", ...). */
SC_API const char* sc_launch_name(const sc_state* state, int64_t frames, int32_t i);
/* Enable/disable CUDA-graph replay (default on). */
SC_API int sc_state_set_graphs(sc_state* state, int32_t enabled);

/* ---- SPEC graph_ir: general DAGs ------------------------------------
 * The reference's model description is a DAG of typed nodes (SPEC NodeKind)
 * joined by ordered (from, to, input port) edges.  Node ids are the array
 * indices (dense integers); edge order into a Sum is its operand order.  Every
 * node has exactly one output edge except FANOUT (`arity`) and SINK (none); every input port
 * (SUM: 0..arity-1, SINK and the others: 0, SOURCE: none) has exactly one incoming edge.
 * GATE and SLICE are builder extensions of SPEC's kinds (the RAVE head, the mean/var split). */
enum sc_gnode_kind {
  SC_G_SOURCE = 0,         /* Source; out_channels = channels (0: the in_channels argument)   */
  SC_G_SINK = 1,           /* Sink                                                            */
  SC_G_CONV = 2,           /* Conv{kernel, stride, dilation, padding}        kernels.cpp:73  */
  SC_G_ZERO_UPSAMPLE = 3,  /* ZeroUpsample{factor}                           kernels.cpp:106 */
  SC_G_ACTIVATION = 4,     /* Activation{kind}                               kernels.cpp:119 */
  SC_G_DELAY = 5,          /* Delay{samples >= 0}     */
  SC_G_SUM = 6,            /* Sum{arity >= 2}: in_0 + in_1 + ... in port order                */
  SC_G_FANOUT = 7,         /* Fanout{arity >= 2}                                              */
  SC_G_GATE = 8,           /* extension: y[c] = tanh(x[c]) * sigmoid(x[c + C/2])              */
  SC_G_SLICE = 9           /* extension: keep channels [slice_begin, slice_begin+slice_count) */
};

typedef struct sc_gnode {
  int32_t kind;          /* enum sc_gnode_kind */
  int32_t in_channels;   /* CONV: M */
  int32_t out_channels;  /* CONV: N;  SOURCE: channels (0 = the in_channels argument) */
  int32_t taps;          /* CONV: K */
  int32_t stride;        /* CONV: S */
  int32_t dilation;      /* CONV: d */
  int64_t pad_left;      /* CONV: PaddingSpec{left,right} (tensor.hpp:90-95) */
  int64_t pad_right;
  int64_t shift;         /* CONV: right pad already folded into the left pad by causalize —
                            the output delay the rewrite introduced (ledger R) */
  int32_t factor;        /* ZERO_UPSAMPLE: s */
  int32_t act;           /* ACTIVATION: enum sc_act */
  float alpha;           /* ACTIVATION: leaky_relu slope */
  int32_t arity;         /* SUM / FANOUT */
  int64_t samples;       /* DELAY: d, at the node's native rate */
  int64_t weight_offset; /* CONV: float offset of weights[N][M][K] then bias[N] */
  int32_t slice_begin;   /* SLICE */
  int32_t slice_count;   /* SLICE */
  int32_t hint;          /* CONV: enum sc_hint */
  int32_t inserted;      /* DELAY: 1 if inserted by causalize (D_a or A_i), else 0 */
} sc_gnode;

typedef struct sc_edge {
  int32_t from;          /* producing node id */
  int32_t to;            /* consuming node id */
  int32_t port;          /* input port of `to` */
} sc_edge;

/* SPEC validate: returns SC_OK iff every GraphIR invariant holds, else
 * CycleDetected / ChannelMismatch / RateMismatchAtSum / DanglingNode / MalformedGraph /
 * InvalidArgument / SchemaError naming the offending node id.  edge_rates (optional,
 * [n_edges][2]) receives the RateMap: edge rate num/den relative to the Source. */
SC_API int sc_graph_validate(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                             int32_t n_edges, int32_t in_channels, int64_t* edge_rates,
                             int32_t* out_channels);
/* SPEC compression_ratio: the streaming buffer granularity — the lcm of
 * every edge rate's denominator (= the denominator of the minimum rate ratio on any
 * Source->Sink path for the stride / upsample products SPEC lists). */
SC_API int sc_graph_compression_ratio(const sc_gnode* nodes, int32_t n_nodes,
                                      const sc_edge* edges, int32_t n_edges,
                                      int32_t in_channels, int64_t* ratio);
/* SPEC receptive_field: past / future extents in input samples by interval
 * propagation (Conv with padding (L,R) adds its span, Delay shifts, Sum / Fanout take the
 * union); extents are rounded up to whole input samples, future is clamped at 0.  An output
 * frame of a stride-S conv stands at the last input frame it consumes (streaming emits it
 * then), so a streamable strided conv (pad >= span - S, all on the left) has future 0. */
SC_API int sc_graph_receptive_field(const sc_gnode* nodes, int32_t n_nodes,
                                    const sc_edge* edges, int32_t n_edges, int32_t in_channels,
                                    int64_t* past, int64_t* future);
/* SPEC causalize as a graph-to-graph rewrite: every Conv pad (L,R) becomes
 * (L+R, 0) with shift += R; Delay(D_a) nodes (Eq. 2) are inserted before strided convs and
 * Delay(A_i) nodes (branch_alignment) on Sum inputs; ids of original nodes are kept, new
 * Delay nodes are appended.  Caps are the capacities of the output arrays (n_nodes + n_edges
 * nodes and 2 x n_edges edges always suffice).  latency = total latency in input samples. */
SC_API int sc_graph_causalize(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                              int32_t n_edges, int32_t in_channels, sc_gnode* out_nodes,
                              int32_t node_cap, int32_t* n_out_nodes, sc_edge* out_edges,
                              int32_t edge_cap, int32_t* n_out_edges, int64_t* latency);
/* SPEC latency_of: NotCausal if the graph's future receptive field is > 0,
 * else its Sink cumulated delay in input samples.  The ledger counts the delay
 * causalize introduces — conv R + shift, and Delay nodes marked `inserted` — but not a Delay
 * of the model itself, which shifts the original and the causalized graph alike (counting it
 * would break offline_run(causalize(g)) == shift(offline_run(g), latency)). */
SC_API int sc_graph_latency(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                            int32_t n_edges, int32_t in_channels, int64_t* samples);
/* SPEC mac_count: exact multiply-accumulates of an offline run over
 * `input_samples` — sum over Conv nodes of out_len x N x M x K, the reference's literal
 * arithmetic (a Conv after a ZeroUpsample counts its zero-stuffed MACs; the GPU's polyphase
 * form skips them, sc_plan_macs_per_sample).  input_samples should be a multiple of the
 * compression ratio (out_len = input_samples x the conv's output rate, rounded down). */
SC_API int sc_graph_mac_count(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                              int32_t n_edges, int32_t in_channels, int64_t input_samples,
                              int64_t* macs);
/* sc_plan_create for a DAG: validate + causalize + lower to the fused cached-conv program.
 * ZeroUpsample must feed a stride-1, dilation-1 Conv (lowered to a polyphase ConvTranspose);
 * a Sum becomes the residual epilogue of a conv branch when one operand is a conv output
 * with nothing else reading it, else one SIMT sum launch; Delays become read offsets. */
SC_API int sc_plan_create_graph(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                                int32_t n_edges, const float* weights_host, int64_t n_weights,
                                int32_t in_channels, int32_t precision, int32_t device,
                                sc_plan** out);

/* ---- SPEC model_io: JSON manifest + raw little-endian f32 blob --------
 * Manifest schema: docs in INTEGRATION.md §model_io.  `blob_path` NULL = the manifest path
 * with its extension replaced by ".bin" (paired files share a basename).
 * Errors: VersionMismatch, CorruptBlob (blob size / weight ranges), SchemaError with the JSON
 * path of the offending value, plus every sc_graph_validate error. */
typedef struct sc_model sc_model;
SC_API int sc_model_load(const char* manifest_path, const char* blob_path, sc_model** out);
/* Arrays owned by the model (valid until sc_model_destroy). */
SC_API int sc_model_graph(const sc_model* model, const sc_gnode** nodes, int32_t* n_nodes,
                          const sc_edge** edges, int32_t* n_edges, const float** weights,
                          int64_t* n_weights, int32_t* in_channels);
SC_API int sc_model_destroy(sc_model* model);
SC_API int sc_model_save(const char* manifest_path, const char* blob_path, const sc_gnode* nodes,
                         int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                         const float* weights, int64_t n_weights, int32_t in_channels);

/* ---- SPEC baseline_ola: overlap-add over the non-causal graph ---------
 * Chunks x[i*hop : i*hop + chunk] (hop = chunk x (1 - overlap/100)) are each run OFFLINE through
 * the unmodified graph (original pads, zero state: offline_run), multiplied by the
 * ratio-scaled window and summed at offsets i*hop; the output is trimmed to the input length.
 * All chunks of all streams run batched on the GPU.  overlap_pct in {0, 25, 50}; chunk and hop
 * must be multiples of the compression ratio (ChunkTooSmall below it).                     */
typedef struct sc_ola sc_ola;
SC_API int sc_ola_create(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                         int32_t n_edges, const float* weights_host, int64_t n_weights,
                         int32_t in_channels, int32_t precision, int32_t device, int64_t chunk,
                         int32_t overlap_pct, int32_t n_streams, int64_t max_frames, sc_ola** out);
/* d_in [n_streams][in_channels][frames] -> d_out [n_streams][out_channels][frames x sink];
 * frames >= chunk, a multiple of the hop, <= max_frames.  Asynchronous on `stream`. */
SC_API int sc_ola_process(sc_ola* ola, const float* d_in, float* d_out, int64_t frames, void* stream);
SC_API int sc_ola_destroy(sc_ola* ola);
/* Lowering summary of the OLA's offline program (valid until sc_ola_destroy). */
SC_API const char* sc_ola_describe(const sc_ola* ola);
/* hann_window: 50 -> sin^2(pi n / N); 25 -> flat top with sin^2 quarter lobes
 * (SPEC.md:350 decision, COLA at hop 3N/4); 0 -> rectangular.  w: N floats (computed in double). */
SC_API int sc_ola_window(int64_t n, int32_t overlap_pct, float* w);
/* redundancy_factor: samples pushed through the network per output sample. */
SC_API double sc_ola_redundancy(int32_t overlap_pct);

/* ---- SPEC metrics_bench fidelity scores, batches of device signals ------
 * ref / test: [n_signals][length] fp32 device.  Any of the outputs may be NULL.
 *   l_s: spectral distance, Eq. 3 (n_fft 256/512/1024, hop n_fft/4, Hann, log(|S|+1), L2 over
 *        frames x bins divided by the frame count, summed over scales; cuFFT)
 *   l_w: Euclidean distance ||x - y||_2, Eq. 4
 *   l_c: normalized correlation; ZeroEnergy (and NaN) when a signal has no energy.
 * Synchronous: returns after the host outputs are written. */
SC_API int sc_fidelity(const float* d_ref, const float* d_test, int32_t n_signals, int64_t length,
                       double* l_s, double* l_w, double* l_c, void* stream);
/* best_lag: argmax over lag in [0, max_lag] of correlation(ref[0:T-lag],
 * test[lag:T]) per signal.  Synchronous. */
SC_API int sc_best_lag(const float* d_ref, const float* d_test, int32_t n_signals, int64_t length,
                       int32_t max_lag, int64_t* lags, void* stream);

/* ---- tensor_core ops on device batches (kernels.hpp:16-32) ----------------------------- */
/* conv1d (kernels.cpp:73-104) over a batch: x [batch][M][L] -> y [batch][N][Lout],
 * Lout = (L - ((K-1)d+1))/S + 1 (kernels.cpp:46-49).  w/b device, reference layout.      */
SC_API int sc_conv1d(const float* d_x, int32_t batch, int32_t in_channels, int64_t length,
              const float* d_w, const float* d_b, int32_t out_channels, int32_t taps,
              int32_t stride, int32_t dilation, float* d_y, void* stream);
SC_API int64_t sc_conv_output_length(int64_t in_len, int32_t taps, int32_t stride, int32_t dilation);

/* ---- PQMF filter bank (not in the reference: builder-defined, parity unpinned) ---------- */
/* Kaiser-windowed lowpass prototype (taps), cosine-modulated into `bands` analysis and
 * synthesis filters, written in the sc_node conv weight layout:
 *   analysis : CONV  M=1, N=bands, K=taps, S=bands, pad (taps-bands, 0)  -> [bands][1][taps]
 *   synthesis: CONVT M=bands, N=1,  K=taps, S=bands, pad (taps-1, 0)     -> [1][bands][taps]
 * Each array is followed by a zero bias.  Computed in double, rounded once to fp32.      */
SC_API int sc_pqmf_filters(int32_t bands, int32_t taps, float* analysis, float* synthesis,
                    double* prototype);

#ifdef __cplusplus
}
#endif
#endif /* STREAMCONV_B200_H */
