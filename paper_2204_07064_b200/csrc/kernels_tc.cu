// kernels_tc.cu — the dense cached-conv on the 5th-gen tensor cores (sm_100a).
//
// Implicit GEMM, output tiles of BM=128 rows (stream x time) by BN output channels:
//   D[m][n] = sum_{q,c} A[m][(q,c)] * W[n][(q,c)]
// where A rows are the cached-padding window of the input buffer (rows = frames, or S-frame
// super-rows for a stride-S conv).  Every (tap, 32-channel block) K-slab of A is a plain box of
// the frame-major buffer, so TMA loads it directly — the "im2col" is free.
//
// fp32-accurate "3xTF32": kind::tf32 consumes only the top 19 bits of each operand, so every
// operand x is split x = hi + lo with hi = x & 0xffffe000 (exactly representable in tf32) and
// lo = x - hi (exact in fp32), and D += A_lo W_hi + A_hi W_lo + A_hi W_hi (the dropped A_lo W_lo
// term is ~2^-22 relative).  Weight hi/lo planes are prepared once at plan time; the
// activation split (and the fused pre-activation LeakyReLU/tanh) is done by the transform
// warps between the TMA landing and the MMA issue, which store A hi / lo into TMEM: all three
// MMAs take A from TMEM, so the only shared-memory operand traffic is the weight tile (shared
// memory bandwidth, not the tensor core, bounded the all-smem form).
//
// The tensor core accumulates in fp32 with truncation, so long K loops drift (measured: ~4e-5
// x RMS per layer at K=384..1536).  The MMA therefore accumulates only CK K-blocks (a chunk)
// into one of two TMEM buffers, and the drain warps add each chunk into fp32 registers with
// round-to-nearest adds (fixed order, independent of T and of the stream count), which keeps
// the path at FFMA-level accuracy at any depth.
//
// Persistent: grid = #SMs, static tile striding; the TMA/transform/MMA pipeline runs across
// tile boundaries and the drain/epilogue of tile t overlaps the MMAs of tile t+1.
// Warp roles (480 threads): w0 TMA producer | w1 TMEM alloc + single-thread MMA issuer |
// w2 epilogue I/O (residual tile TMA-loaded into the staging buffer once the previous output
// store has read it; output tile TMA-stored from staging) | w3..w6 transform | w7..w14 drain +
// epilogue (TMEM lane quarter = warp % 4, column half = (warp - 7) / 4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "kernels_tc.hpp"

namespace scb {

namespace {

__device__ long long g_tc_trace[32 * 256];  // SC_TC_DEBUG & 32: per-K-block timestamps of CTA 0

__device__ __forceinline__ long long clk() { return clock64(); }  // SM cycles (per-SM counter)

// Experiment hooks (per-slab trace timestamps, MMA / prefetch switches: TcParams::debug) are
// compiled in only with -DSC_TC_EXPERIMENTS=1 — even untaken, their branches cost the hot
// loops measurable time.
#ifndef SC_TC_EXPERIMENTS
#define SC_TC_EXPERIMENTS 0
#endif
#define TC_DBG(p) (SC_TC_EXPERIMENTS ? (p).debug : 0)

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 per 128-byte swizzled row
constexpr uint32_t A_TILE = BM * BK * 4;  // 16 KB
constexpr int NUM_THREADS = 480;
constexpr int IO_WARP = 2;    // residual TMA loads + output TMA stores
constexpr int XF_WARP0 = 3;   // transform warps 3..6 (3..10: two sets, X2)
constexpr int EP_WARP0 = 7;   // drain/epilogue warps 7..14 (11..18, X2)
// X2 (3xFP16 non-window tiles): two sets of four transform warps take alternate K-slabs — one
// set of four (one warp per SM sub-partition) could not split a slab as fast as kind::f16 MMAs
// consume it (measured ~0.9k cycles per slab vs 384 cycles of MMA)
// X2 also has its own A-unit producer warp (EP0 + 8), so the input loads run ahead of the W ring.
template <bool X2> struct Roles {
  static constexpr int XF0 = X2 ? 4 : XF_WARP0;  // X2: w0 W | w1 MMA | w2 I/O | w3 A units
  static constexpr int NXF = X2 ? 8 : 4;
  static constexpr int EP0 = XF0 + NXF;
  static constexpr int AW_WARP = 3;
  static constexpr int NT = (EP0 + 8) * 32;
};

template <uint32_t N> __device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N> __device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

// packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): same round-to-nearest results as
// the scalar forms, half the instructions
__device__ __forceinline__ void ffma2_acc(float& a0, float& a1, float v0, float v1, float f) {  // a += v * f
  asm("{\n\t.reg .b64 A, V, F;\n\tmov.b64 A, {%0, %1};\n\tmov.b64 V, {%2, %3};\n\tmov.b64 F, {%4, %4};\n\t"
      "fma.rn.f32x2 A, V, F, A;\n\tmov.b64 {%0, %1}, A;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(v0), "f"(v1), "f"(f));
}
__device__ __forceinline__ void fadd2_acc(float& a0, float& a1, float v0, float v1) {  // a += v
  asm("{\n\t.reg .b64 A, V;\n\tmov.b64 A, {%0, %1};\n\tmov.b64 V, {%2, %3};\n\t"
      "add.rn.f32x2 A, A, V;\n\tmov.b64 {%0, %1}, A;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(v0), "f"(v1));
}
__device__ __forceinline__ float2 fmul2s(float x0, float x1, float f) {  // x * f
  float2 r;
  asm("{\n\t.reg .b64 X, F, R;\n\tmov.b64 X, {%2, %3};\n\tmov.b64 F, {%4, %4};\n\t"
      "mul.rn.f32x2 R, X, F;\n\tmov.b64 {%0, %1}, R;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(x0), "f"(x1), "f"(f));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {  // a - b
  float2 r;
  asm("{\n\t.reg .b64 A, B, R;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\t"
      "sub.rn.f32x2 R, A, B;\n\tmov.b64 {%0, %1}, R;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// 3xFP16 split of a (scaled) pair: hi = fp16_rn(t) (one packed conversion), lo = fp16_rn(t -
// float(hi)) — t - hi is exact in fp32, so hi + lo carries >= 22 significant bits of t, as tf32
// hi + lo does.  The unpack of hi runs as HADD2.F32 on the FMA-class pipe: per pair two ALU-pipe
// conversions and three FMA-pipe operations.  (Forms tried before: an integer round or mask of
// the fp32 bits for hi — two more ALU-pipe operations per pair, and the ALU pipe, which issues a
// warp instruction every other cycle, is the transform's busiest unit (ncu: "math pipe throttle"
// on a quarter of its samples); cvt.f32.f16 for the unpack — the conversion unit at 126% of peak;
// a Veltkamp split, c t - (c t - t) — folded to t by ptxas.)  SC_SPLIT_MASK=1 builds the mask form.
// hi is exact in fp16 down to 2^-14; below that (< 2^-28 of the row max after scaling) it rounds
// to fp16 subnormals and lo picks up the remainder — a fixed function of the row like the scale.
#ifndef SC_SPLIT_MASK
#define SC_SPLIT_MASK 0
#endif
__device__ __forceinline__ void split_f16x2(float2 t, uint32_t& h, uint32_t& l) {
#if SC_SPLIT_MASK
  float2 hi;
  hi.x = __uint_as_float(__float_as_uint(t.x) & 0xFFFFE000u);
  hi.y = __uint_as_float(__float_as_uint(t.y) & 0xFFFFE000u);
  const __half2 h2 = __floats2half2_rn(hi.x, hi.y);
#else
  const __half2 h2 = __floats2half2_rn(t.x, t.y);
  const float2 hi = __half22float2(h2);
#endif
  const float2 lo = fsub2(t, hi);
  const __half2 l2 = __floats2half2_rn(lo.x, lo.y);
  h = *reinterpret_cast<const uint32_t*>(&h2);
  l = *reinterpret_cast<const uint32_t*>(&l2);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Waits off the critical path back off with nanosleep between polls: a failed try_wait returns
// within ~20 cycles, so a spinning warp takes one issue slot in ten from the transform / drain
// warps of its SM sub-partition (ncu source counters: 17% of all executed instructions were
// wait loops).  ns = 0 keeps the plain spin.
#ifndef SC_SLEEP_IO
#define SC_SLEEP_IO 128    // epilogue I/O lane: once per tile
#endif
#ifndef SC_SLEEP_PROD
#define SC_SLEEP_PROD 64   // TMA producers waiting for a free ring slot
#endif
#ifndef SC_SLEEP_DRAIN
#define SC_SLEEP_DRAIN 32  // drain warps waiting for a chunk (two more chunk buffers of slack)
#endif
#ifndef SC_SLEEP_XF
#define SC_SLEEP_XF 32     // transform warps waiting for input rows to land
#endif
template <uint32_t NS> __device__ __forceinline__ void mbar_wait_bo(uint64_t* bar, uint32_t parity) {
  if constexpr (NS == 0) {
    mbar_wait(bar, parity);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "nanosleep.u32 %2;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(NS)
        : "memory");
  }
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_w(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_w(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                              int c2) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// K-major, 128B-swizzled canonical layout: 8-row x 128 B atoms stacked at SBO = 1024 B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);  // start address
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
  d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// K-major, 64B-swizzled canonical layout (bf16 rows of 32 elements): atoms of 8 rows x 64 B.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;  // SBO: 8 rows x 64 B
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;         // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// A operand from TMEM (lanes = M rows, 32-bit columns = K)
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

// Warp-collective forms: the whole warp runs the issue loop in uniform control flow (so the
// descriptors live in uniform registers) and elect.sync picks the one issuing lane.  Issuing
// from a lane-0-only branch instead costs an R2UR waterfall per tcgen05.mma (~80 cycles).
__device__ __forceinline__ void mma_tf32_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One K-slab of the 3xFP16 product (two K = 16 steps, A hi | lo from TMEM): the corrections
// A_lo W_hi, A_hi W_lo of both steps, then A_hi W_hi — six MMAs under one elected lane.
__device__ __forceinline__ void mma_f16x3_slab_w(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t bh0, uint64_t bh1,
                                                 uint64_t bl0, uint64_t bl1, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %9, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %8, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %8, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %4, %8, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %6, %8, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %8, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %4, %8, t;\n\t}" ::"r"(d),
      "r"(ahi), "r"(alo), "l"(bh0), "l"(bh1), "l"(bl0), "l"(bl1), "r"(0), "r"(idesc), "r"(acc0), "r"(alo + 8),
      "r"(ahi + 8)
      : "memory");
}

// The same six MMAs with both operands in shared memory (window tiles: A = fp16 hi / lo window
// planes at a tap's row offset): descriptors of the first K = 16 step; the second step's start 32
// bytes (2 descriptor address units) further.  One elected lane, one asm block: issuing the six
// MMAs one call at a time cost ~120 uniform-datapath instructions per K-slab in the issuing warp
// (descriptor rebuilds, an elect per MMA) — more than the 192 cycles the N = 64 MMAs take.
__device__ __forceinline__ void mma_f16x3_slab_ss_w(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                                    uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t.reg .b64 ah1, al1, bh1, bl1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "add.u64 ah1, %1, 2;\n\t"
      "add.u64 al1, %2, 2;\n\t"
      "add.u64 bh1, %3, 2;\n\t"
      "add.u64 bl1, %4, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %4, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], al1, bh1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ah1, bl1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ah1, bh1, %5, t;\n\t}" ::"r"(d),
      "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc0)
      : "memory");
}

__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t warp_uniform(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// tanh is kept out of line: inlining it into the fully unrolled transform and epilogue loops
// bloats the kernel past the instruction cache (measured: 4-16 us epilogues).
__device__ __noinline__ float tanh_ool(float v) { return tanhf(v); }
// The gated head's tanh(a) sigmoid(g) from two hardware exponentials and two approximate
// reciprocals: tanh(a) = (e^2a - 1) / (e^2a + 1) with a clamped to +-15 (tanh(15) = 1 - 2e-13)
// — and, below |a| = 0.1 where e^2a - 1 cancels, the odd series a - a^3/3 + 2a^5/15 - 17a^7/315
// (next term 2e-11) — times 1 / (1 + e^-g).  ex2.approx and the reciprocal are accurate to 2
// ulp: relative error ~1e-6 at every signal level (quiet streams keep their relative accuracy),
// against ~170 instructions per output for the tanhf / expf / IEEE-division form (the head was
// the launch with the most executed instructions of the cfg5 step).  e^-g -> inf gives 0, the
// gate's limit.
__device__ __forceinline__ float gate_fast(float a, float g) {
  const float ac = fminf(fmaxf(a, -15.f), 15.f);
  const float e2 = __expf(2.f * ac), eg = __expf(-g);
  const float a2 = a * a;
  const float series = a * fmaf(a2, fmaf(a2, fmaf(a2, -17.f / 315.f, 2.f / 15.f), -1.f / 3.f), 1.f);
  const float th = fabsf(a) < 0.1f ? series : __fdividef(e2 - 1.f, e2 + 1.f);
  return th * __fdividef(1.f, 1.f + eg);
}

// LeakyReLU / identity as one branch-free form (slope 1 = identity): no call, no spill
__device__ __forceinline__ float act_lin(float v, float slope) { return v < 0.f ? slope * v : v; }
__device__ __forceinline__ float slope_of(int kind, float alpha) { return kind == ACT_LRELU ? alpha : 1.f; }

__device__ __forceinline__ float act_apply(float v, int kind, float alpha) {
  if (kind == ACT_LRELU) return v < 0.f ? alpha * v : v;
  if (kind == ACT_TANH) return tanh_ool(v);
  return v;
}

// fp32 (3xTF32) stage: A raw | W hi | W lo, K-major SW128 (32 fp32/row); A hi / lo go to
//                      TMEM (per-stage columns).
// bf16 stage:          A raw fp32 (SW128) | A bf16 (SW64, 32 bf16/row) | W bf16 (SW64).
// window stage (WIN, fp32, narrow tiles): the ring holds only W hi | W lo; two window slots
// hold the 128 + halo input rows of one 32-channel block as A hi and A lo (SW128), computed
// once and read by the SS-MMAs of every tap at a row offset (q x tap_rows x 128 B: the
// swizzle follows absolute address bits, so a descriptor may start at any 128 B row —
// tools/desc_rowshift_test.cu).
// The window kernels' weight region (112 KB) holds either a ring of K-slab tiles or, when
// the layer's whole weight (hi + lo) fits, all of it — loaded once per CTA (p.wres).
constexpr int WIN_ROWS = 144;     // fp32 windows: 128 + halo (<= 16)
constexpr int WIN_ROWS_BF = 192;  // bf16 windows of narrow tiles: 128 + halo (<= 64)
constexpr uint32_t WREG = 112 * 1024;
constexpr uint32_t WREG_H = 56 * 1024;  // 3xFP16 windows: fp16 hi + lo weight planes are half the bytes
// 3xFP16 (HF): per-row power-of-two scale exponents, one byte per (32-channel row, K-slab):
// a ring of RS_RING slabs x 128 rows (non-window) or RS_WIN windows x WROWS rows (window mode),
// deep enough that the transform never overwrites an entry the drain has not read yet
// (transform of slab g implies the drain finished slab g - STAGES - NB; see HF below)
constexpr int RS_RING = 32;
constexpr int AW_ROWS = 192;  // X2 A units: G x (R + halo) rows of one 32-channel block (24 KB)
constexpr int RS_WIN = 16;
template <int BN, int STAGES, bool BF = false, bool WIN = false, int IOB = 0, bool HF = false>
struct TcSmem {
  static constexpr uint32_t B_TILE = (BF || HF) ? BN * BK * 2 : BN * BK * 4;
  // X2 (3xFP16 non-window): the stage ring holds only W hi | lo; the input rows come through a
  // separate ring of A units (per-slab boxes, or per 32-channel-block windows of every tap)
  static constexpr bool X2 = HF && !WIN;
  static constexpr uint32_t STAGE = (WIN || X2) ? (BF ? B_TILE : 2 * B_TILE) : BF ? A_TILE + B_TILE : A_TILE + 2 * B_TILE;
  // window slots: fp32 = A hi + A lo (SW128); bf16 = the raw fp32 rows + their bf16 copy (SW64);
  // 3xFP16 = the raw fp32 rows, converted in place to fp16 hi | lo planes (SW64)
  static constexpr int AST = WIN ? (BF ? 3 : HF ? 4 : 2) : X2 ? 3 : 0;
  // bf16 windows hold 128 + 64 rows when they fit three slots next to the staging tile (narrow
  // tiles, or bf16 input rows: a raw bf16 row is half the size)
  static constexpr bool ABF = BF && (IOB & 1);
  static constexpr int WROWS = (BF && (BN < 128 || ABF)) ? WIN_ROWS_BF : WIN_ROWS;
  static constexpr uint32_t WIN_SLOT = BF ? WROWS * BK * ((ABF ? 2 : 4) + 2)
                                       : X2 ? AW_ROWS * BK * 4 : HF ? WROWS * BK * 4 : 2 * WROWS * BK * 4;
  static constexpr uint32_t STAGING = BM * BN * 4;  // residual-in / output-out tile, 32-col SW128 slabs
  // 3xFP16 BN = 128 windows: a W ring of STAGES K-slab tiles (never resident); BN <= 64: the
  // 56 KB weight region (ring or the whole weight)
  static constexpr uint32_t WBYTES =
      (WIN && !BF) ? (HF ? (BN == 128 ? STAGES * STAGE : WREG_H) : WREG) : STAGES * STAGE;
  static constexpr uint32_t RSB = HF ? (WIN ? RS_WIN * WROWS : RS_RING * BM) : 0;
  static constexpr uint32_t BYTES =
      WBYTES + AST * WIN_SLOT + STAGING + 1024 /*barriers*/ + 8192 /*bias*/ + RSB + 1024;
  static_assert(!WIN || BF || (HF && BN == 128) || STAGES * STAGE <= (HF ? WREG_H : WREG),
                "window ring fits the weight region");
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// float offset of (row, col) inside a staging tile of 32-column 128B-swizzled slabs
// bf16 element offset of (row, col) inside a staging tile of 32-column 64B-swizzled slabs
__device__ __forceinline__ int stg_off_b(int row, int col) {
  const int slab = col >> 5, c = col & 31;
  return slab * (BM * 32) + row * 32 + ((((c >> 3) ^ ((row >> 1) & 3))) << 3) + (c & 7);
}
__device__ __forceinline__ int stg_off(int row, int col) {
  const int slab = col >> 5, c = col & 31;
  return slab * (BM * 32) + row * 32 + ((((c >> 2) ^ (row & 7))) << 2) + (c & 3);
}

struct TileCoord {
  int s0, i0, n0;
};

__device__ __forceinline__ TileCoord tile_coord(const TcParams& p, int tile, int n_tiles_n, int BN) {
  const int mt = tile / n_tiles_n;
  const int nt = tile - mt * n_tiles_n;
  TileCoord tc;
  tc.n0 = nt * BN;
  if (p.G == 1) {
    tc.s0 = mt / p.tiles_per_stream;
    tc.i0 = (mt - tc.s0 * p.tiles_per_stream) * p.R;
  } else {
    tc.s0 = mt * p.G;
    tc.i0 = 0;
  }
  return tc;
}

// IOB (bf16 plans): bit 0 = the input buffer holds bf16, bit 1 = the output (and residual)
// buffer holds bf16 — compile-time, so each instance carries only its own load / store paths
//
// HF (fp32 plans, "3xFP16"): the same three-product split as 3xTF32, in fp16 — kind::f16 runs at
// twice the kind::tf32 rate and the weight planes are half the bytes.  fp16 has tf32's 11-bit
// significand but only a 5-bit exponent, so every operand row is block-scaled by a power of two
// first (exact): the transform scales each (row, 32-channel K-slab) so its largest |a| lands in
// [2^14, 2^15), splits a = hi + lo (hi = fp16_rn(a), lo = fp16_rn(a - hi): ~22 significant bits,
// as tf32 hi + lo), and records the unscale exponent; weights carry one power-of-two scale per
// layer (plan time).  Each K-slab is its own chunk accumulator (CK = 1), so the drain multiplies
// the chunk by the row's exact 2^-(s + s_w) as it adds it (one fma: the product is exact).  The
// scale depends only on the row's own 32 values: identical in window and non-window mode, for
// any tile geometry (bit-identity across buffer partitions).
template <int BN, int STAGES, int CK, bool BF, bool WIN, int IOB, bool CH, bool HF>
__global__ void __launch_bounds__(Roles<HF>::NT, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
                   const __grid_constant__ CUtensorMap tmap_out, const __grid_constant__ CUtensorMap tmap_res,
                   const TcParams p) {
  using L = TcSmem<BN, STAGES, BF, WIN, IOB, HF>;
  static_assert(!HF || (!BF && !CH && CK == 1), "3xFP16: fp32 plans, unchained, one K-slab per chunk");
  constexpr bool X2 = L::X2;  // 3xFP16 non-window layout (A units + W ring)
  constexpr bool RX = HF;     // 3xFP16 (window or not): warpgroup roles, two transform sets
  constexpr int EP0 = Roles<RX>::EP0;
  constexpr int NT = Roles<RX>::NT;
  constexpr bool ABF = BF && (IOB & 1);  // input rows are bf16
  constexpr bool OBF = BF && (IOB & 2);  // output / residual rows are bf16
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by an offset from the __shared__ array (not integer pointer math), so
  // the compiler keeps the shared address space: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* wins = smem + L::WBYTES;
  float* stg = reinterpret_cast<float*>(wins + L::AST * L::WIN_SLOT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wins + L::AST * L::WIN_SLOT + L::STAGING);
  uint64_t* full = bars;
  uint64_t* xform = bars + STAGES;
  uint64_t* empty = bars + 2 * STAGES;
  uint64_t* res_full = bars + 3 * STAGES + 4;
  uint64_t* stg_written = bars + 3 * STAGES + 5;
  uint64_t* stg_free = bars + 3 * STAGES + 6;
  uint64_t* aempty = bars + 3 * STAGES + 8;  // [<= STAGES] TMEM A slots
  uint64_t* wa_full = bars + 4 * STAGES + 8;    // [AST] window rows landed (WIN)
  uint64_t* wa_ready = bars + 4 * STAGES + 12;  // [AST] window hi / lo (bf16 copy) written (WIN)
  uint64_t* wa_empty = bars + 4 * STAGES + 16;  // [AST] window read by the last tap's MMAs (WIN)
  uint64_t* tfull = bars + 4 * STAGES + 20;   // [NB] main chunk accumulated
  uint64_t* tempty = bars + 4 * STAGES + 28;  // [NB] main chunk drained
  uint64_t* wres_full = bars + 4 * STAGES + 36;   // resident weights landed (WIN && p.wres)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * STAGES + 37);
  uint64_t* a2full = bars + 4 * STAGES + 38;   // [<= 4] chained GEMM's A slot written (CH)
  uint64_t* a2empty = bars + 4 * STAGES + 42;  // [<= 4] chained GEMM's A slot read by its MMAs (CH)
  float* sbias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 1024);  // <= 2048 floats
  uint8_t* rsc = reinterpret_cast<uint8_t*>(bars) + 1024 + 8192;  // HF: per-row unscale exponents

  auto a_hi = [&](int s) { return smem + s * L::STAGE; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE + ((WIN || X2) ? 0 : A_TILE); };
  auto b_lo = [&](int s) { return smem + s * L::STAGE + ((WIN || X2) ? 0 : A_TILE) + L::B_TILE; };
  auto b_bf = [&](int s) { return smem + s * L::STAGE + A_TILE; };
  auto win_hi = [&](int sa) { return wins + sa * L::WIN_SLOT; };
  auto win_lo = [&](int sa) { return wins + sa * L::WIN_SLOT + L::WROWS * BK * 4; };  // fp32: A lo
  auto win_bf = [&](int sa) { return wins + sa * L::WIN_SLOT + L::WROWS * BK * (ABF ? 2 : 4); };  // bf16 copy
  auto win_lo16 = [&](int sa) { return wins + sa * L::WIN_SLOT + L::WROWS * BK * 2; };  // HF: fp16 lo plane

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = p.n_kblocks;
  // chained 1x1 conv (CH): nk first-conv K-slabs, then NK2 slabs of the second conv whose A
  // operand the drain writes from the first conv's finished tile
  constexpr int NK2 = CH ? BN / BK : 0;
  const int nkt = nk + NK2;
  const int n_tiles_n = (p.nout + BN - 1) / BN;
  const int n_tiles = p.m_tiles * n_tiles_n;
  // TMEM columns: NB chunk accumulators (BN each) | A ring of TS slots — fp32: A hi (32 cols)
  // + A lo (32 cols) per slot (none in window mode: A is in shared memory); bf16: 16 cols per
  // slot (32 bf16 per row, two per column).  As many chunk accumulators as fit (<= 8), so the
  // MMAs run ahead across a tile-boundary epilogue.
  constexpr int TS = BF ? STAGES : WIN ? 2 : HF ? 4 : BN == 128 ? 2 : (STAGES < 4 ? STAGES : 4);
  static_assert(4 * STAGES + 46 <= 128, "barrier area");
  static_assert(!CH || (BN == 128 && CK == (BF ? 4 : 1) && (BF || !WIN)), "chained conv: BN = 128 (windows: bf16)");
  static_assert(TS >= 2, "TMEM A ring needs two slots");
  static_assert(!X2 || 4 * A_TILE <= L::AST * L::WIN_SLOT, "four per-slab A units fit the unit ring");
  constexpr int OTHER = WIN ? 0 : BF ? 16 * TS : HF ? 32 * TS : 64 * TS;
  // CH: two chunk accumulators + the A ring + the chained GEMM's A slots — fp32: two slots of
  // 64 columns (32 channels hi | lo); bf16: four of 16 (32 channels as bf16 pairs, one per slab)
  constexpr int NS2 = BF ? 4 : 2;
  constexpr int W2 = BF ? 16 : 64;
  // fp32 (SHR): the chained GEMM's A slabs take their turn in the first conv's TMEM A ring
  // (ring positions nk .. nk + 3 of each tile), which leaves room for three chunk accumulators
  constexpr bool SHR = CH && !BF;
  constexpr int NB = CH ? (SHR || WIN ? 3 : 2) : (512 - OTHER) / BN > 8 ? 8 : (512 - OTHER) / BN;
  static_assert(NB >= 2, "two chunk accumulators");
  constexpr uint32_t COLS_USED = NB * BN + OTHER + (CH && !SHR ? NS2 * W2 : 0);
  constexpr uint32_t TMEM_COLS = COLS_USED <= 32 ? 32 : COLS_USED <= 64 ? 64 : COLS_USED <= 128 ? 128
                                 : COLS_USED <= 256 ? 256 : 512;
  static_assert(COLS_USED <= 512, "TMEM budget");
  constexpr uint32_t A_COL = NB * BN;
  constexpr uint32_t A2_COL = NB * BN + OTHER;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xform[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    mbar_init(wres_full, 1);
    for (int a = 0; a < NS2; ++a) {
      mbar_init(&a2full[a], 4);  // the four lane-quarter warps of one drain half
      mbar_init(&a2empty[a], 1);
    }
    mbar_init(res_full, 1);
    mbar_init(stg_written, 8);
    mbar_init(stg_free, 1);
    for (int a = 0; a < STAGES; ++a) mbar_init(&aempty[a], 1);
    for (int a = 0; a < (X2 ? 4 : L::AST > 0 ? L::AST : 1); ++a) {
      mbar_init(&wa_full[a], 1);
      mbar_init(&wa_ready[a], 4);
      mbar_init(&wa_empty[a], X2 ? (p.awin ? 8 : 4) : 1);  // X2: released by the transform warps that read the unit
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_out)) : "memory");
  }
  if ((TC_DBG(p) & 32) && threadIdx.x == 0 && blockIdx.x < 256) {
    g_tc_trace[7 * 256 + blockIdx.x] = clk();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tc_trace[9 * 256 + blockIdx.x] = smid;
  }
  for (int i = threadIdx.x; i < p.nout; i += NT) sbias[i] = p.bias[i];
  if (CH)  // first conv's bias at [0, BN) (p.bias), the chained conv's at [BN, 2 BN)
    for (int i = threadIdx.x; i < BN; i += NT) sbias[BN + i] = p.bias2[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: everything above (barriers, TMEM, bias, tensor-map prefetch)
  // touches only this launch's constants, so it overlaps the previous kernel's tail; the
  // activations it wrote are read only after its grid has completed.  The next launch may start
  // its own prologue as this grid's CTAs retire.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // role bodies shared by the X2 and the classic layouts
  auto role_mma = [&]() {
      // ===================== MMA issuer (whole warp, one elected lane issues) =====================
      {
        const uint32_t tbase = warp_uniform(tmem_base);
        // c_format F32 | a,b format TF32 (2) or BF16 (1) | N >> 3 | M >> 4
        const uint32_t fmt = BF ? 1u : HF ? 0u : 2u;  // HF: F16
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                               (static_cast<uint32_t>(BM >> 4) << 24);
        int g = 0, c = 0, tcount = 0, ga = 0;  // ga: A-ring slab counter (first-conv slabs)
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
          for (int kb = 0; kb < nkt; ++kb, ++g) {
            const int s = g % STAGES;
            const int b = c % NB;
            const bool one2 = CH && p.chain_one && kb >= nk;  // chained GEMM in one accumulator
            const bool chunk_first = one2 ? kb == nk : (kb % CK) == 0;
            const bool chunk_last = one2 ? kb == nkt - 1 : ((kb % CK) == CK - 1) || (kb == nk - 1) || kb >= nk;
            if (chunk_first && c >= NB) mbar_wait(&tempty[b], ((c / NB) + 1) & 1);
            if (CH && kb >= nk) {
              // chained GEMM slab: W from the ring, A (h hi / lo of 32 channels) from the slot
              // the drain wrote; its own chunk accumulator like every first-conv slab
              const int u = tcount * NK2 + (kb - nk), sl = u % NS2;
              mbar_wait(&xform[s], (g / STAGES) & 1);
              mbar_wait(&a2full[sl], (u / NS2) & 1);
              tc_fence_after();
              const uint32_t dmain = tbase + static_cast<uint32_t>(b * BN);
              if (BF) {
                const uint32_t bb = smem_u32(b_bf(s)), at = tbase + A2_COL + W2 * sl;
  #pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  mma_bf16_ts_w(dmain, at + kk * 8, sw64_desc(bb + kk * 32), idesc, (!chunk_first || kk > 0) ? 1u : 0u);
              } else {
                const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
                const uint32_t ahi = tbase + (SHR ? A_COL + 64 * (ga % TS) : A2_COL + W2 * sl), alo = ahi + 32;
  #pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                  mma_tf32_ts_w(dmain, alo + kk * 8, sw128_desc(bh + kk * 32), idesc, (!chunk_first || kk > 0) ? 1u : 0u);
                  mma_tf32_ts_w(dmain, ahi + kk * 8, sw128_desc(bl + kk * 32), idesc, 1u);
                }
  #pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) mma_tf32_ts_w(dmain, ahi + kk * 8, sw128_desc(bh + kk * 32), idesc, 1u);
              }
              if (SHR) {
                mma_commit_w(&aempty[ga % TS]);
                ++ga;
              } else {
                mma_commit_w(&a2empty[sl]);
              }
              mma_commit_w(&empty[s]);
              if (chunk_last) {
                mma_commit_w(&tfull[b]);
                ++c;
              }
              continue;
            }
            mbar_wait(&xform[s], (g / STAGES) & 1);
            if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[3 * 256 + g] = clk();
            tc_fence_after();
            const uint32_t dmain = tbase + static_cast<uint32_t>(b * BN);
            if (BF) {
              // A (bf16 pairs) from this stage's TMEM columns, W from shared memory
              const uint32_t bb = smem_u32(b_bf(s));
              const uint32_t at = tbase + A_COL + 16 * (ga % TS);
  #pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {  // 16 bf16 = 8 TMEM columns / 32 bytes of the 64B row
                const uint32_t acc0 = (!chunk_first || kk > 0) ? 1u : 0u;
                mma_bf16_ts_w(dmain, at + kk * 8, sw64_desc(bb + kk * 32), idesc, acc0);
              }
              mma_commit_w(&aempty[ga % TS]);
            } else if (HF) {
              // fp16 A hi | lo (16 TMEM columns each) from this slab's A slot, W hi / lo planes
              // (SW64) from shared memory; corrections first, then the main product.  X2: the
              // transform does not touch the W stage, so wait for its landing here
              mbar_wait(&full[s], (g / STAGES) & 1);
              const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
              const uint32_t ahi = tbase + A_COL + 32 * (ga % TS), alo = ahi + 16;
              mma_f16x3_slab_w(dmain, ahi, alo, sw64_desc(bh), sw64_desc(bh + 32), sw64_desc(bl), sw64_desc(bl + 32), idesc,
                               chunk_first ? 0u : 1u);
              mma_commit_w(&aempty[ga % TS]);
            } else {
              // A hi / lo from this stage's TMEM columns, W hi / lo from shared memory: the only
              // shared-memory operand traffic is the weight tile (A never re-read from smem).
              // Corrections first (2^-10 of the signal), then the main product, all into this
              // chunk's accumulator: the truncating accumulation meets the large terms only in
              // its last four steps.
              const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
              const uint32_t ahi = tbase + A_COL + 64 * (ga % TS);
              const uint32_t alo = ahi + 32;
              if (!(TC_DBG(p) & 2)) {
  #pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                  const uint32_t acc0 = (!chunk_first || kk > 0) ? 1u : 0u;
                  mma_tf32_ts_w(dmain, alo + kk * 8, sw128_desc(bh + kk * 32), idesc, acc0);
                  mma_tf32_ts_w(dmain, ahi + kk * 8, sw128_desc(bl + kk * 32), idesc, 1u);
                }
              }
  #pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {  // 8 tf32 = 8 TMEM columns / 32 B of the row
                const uint32_t acc0 = (!chunk_first || kk > 0 || !(TC_DBG(p) & 2)) ? 1u : 0u;
                mma_tf32_ts_w(dmain, ahi + kk * 8, sw128_desc(bh + kk * 32), idesc, acc0);
              }
              mma_commit_w(&aempty[ga % TS]);
            }
            ++ga;
            mma_commit_w(&empty[s]);
            if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[11 * 256 + g] = clk();
            if (chunk_last) {
              mma_commit_w(&tfull[b]);
              ++c;
            }
          }
        }
      }
  };
  auto role_io = [&]() {
      // ===================== epilogue I/O (one thread) =====================
      if (lane == 0) {
        const int n_tiles_n2 = n_tiles_n;
        const int out_cols = p.gate ? BN / 2 : BN;
        int tcount = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
          const TileCoord tc = tile_coord(p, tile, n_tiles_n2, BN);
          if (p.res) {  // staging is free (previous store read it): bring this tile's residual in
            const int res_es = OBF ? 2 : 4;  // bytes per residual element (slab = BM x 32 elements)
            mbar_expect_tx(res_full, static_cast<uint32_t>(BN / 32) * 32u * res_es * p.R * p.G);
            for (int k = 0; k < BN / 32; ++k)
              tma_load_3d(&tmap_res, res_full, reinterpret_cast<uint8_t*>(stg) + k * (BM * 32 * res_es),
                          p.res_off + tc.n0 + 32 * k, tc.i0, tc.s0);
            // warm L2 with the next tile's residual: its load is issued only once this tile's
            // output has left staging, so it must not also pay the DRAM latency
            if (tile + static_cast<int>(gridDim.x) < n_tiles && !(TC_DBG(p) & 4)) {
              const TileCoord tn = tile_coord(p, tile + gridDim.x, n_tiles_n2, BN);
              for (int k = 0; k < BN / 32; ++k) tma_prefetch_3d(&tmap_res, p.res_off + tn.n0 + 32 * k, tn.i0, tn.s0);
            }
          }
          mbar_wait_bo<SC_SLEEP_IO>(stg_written, tcount & 1);
          const int oc0 = p.gate ? tc.n0 / 2 : tc.n0;
          for (int k = 0; k < (out_cols + 31) / 32; ++k)
            tma_store_3d(&tmap_out, reinterpret_cast<uint8_t*>(stg) + k * (BM * 32 * (OBF ? 2 : 4)), oc0 + 32 * k,
                         tc.i0, tc.s0);
          bulk_commit();
          bulk_wait_read0();
          mbar_arrive(stg_free);
        }
        bulk_wait0();
      }
  };
  auto role_drain = [&]() {
      // ===================== drain + epilogue (w7..w14; X2: w11..w18) =====================
      constexpr int COLS = BN / 2;
      const int quarter = warp & 3;
      const int half = (warp - EP0) >> 2;
      const int r = quarter * 32 + lane;  // tile row == TMEM lane
      const int col0 = half * COLS;
      const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + col0;
      float acc[COLS];
  #pragma unroll
      for (int u = 0; u < COLS; ++u) acc[u] = 0.f;
      int c = 0, tcount = 0;
      int cb_ = 0, cph = 0;  // HF: chunk buffer c % NB and its phase (c / NB) & 1, kept incrementally
      const int taps_w = nk / p.cblocks;  // window mode (HF): chunk kb = (32-channel block, tap)
      const uint8_t* rs_row = rsc + r;     // HF: this row's scale bytes
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
        int wq = 0, wu = tcount * p.cblocks;  // HF window: this chunk's tap and window count
        if (HF) {  // the bias is the accumulator's start value (one load per tile, not per chunk)
  #pragma unroll
          for (int u = 0; u < COLS; u += 4) {
            const float4 bv = *reinterpret_cast<const float4*>(sbias + tc.n0 + col0 + u);
            acc[u] = bv.x, acc[u + 1] = bv.y, acc[u + 2] = bv.z, acc[u + 3] = bv.w;
          }
        }
#pragma unroll 1
        for (int kb = 0; kb < nkt; ++kb) {
          const bool one2 = CH && p.chain_one && kb >= nk;
          const bool chunk_last = one2 ? kb == nkt - 1 : ((kb % CK) == CK - 1) || (kb == nk - 1) || kb >= nk;
          if (!chunk_last) continue;
          const bool first = (kb / CK) == 0 || kb == (one2 ? nkt - 1 : nk);  // + the chained conv's first chunk
          const int boff = (CH && kb >= nk) ? BN : 0;     // its bias sits at sbias[BN, 2 BN)
          const int b = HF ? cb_ : c % NB;
          mbar_wait_bo<SC_SLEEP_DRAIN>(&tfull[b], HF ? cph : (c / NB) & 1);
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && c < 256 && warp == EP0 && lane == 0) g_tc_trace[5 * 256 + c] = clk();
          tc_fence_after();
          float f = 1.f;  // HF: this (row, K-slab)'s exact unscale 2^-(s + s_w)
          if (HF) {
            uint32_t eb;
            if (WIN) {
              eb = rs_row[(wu % RS_WIN) * L::WROWS + wq * p.a_tap_rows];
              if (++wq == taps_w) wq = 0, ++wu;
            } else {
              eb = rs_row[(c % RS_RING) * BM];
            }
            f = __uint_as_float(eb << 23);
            if (++cb_ == NB) cb_ = 0, cph ^= 1;
          }
          // main chunk, 32 columns per TMEM load (16 for the narrowest tiles)
          constexpr int LDC = COLS >= 32 ? 32 : 16;
  #pragma unroll
          for (int cc = 0; cc < COLS; cc += LDC) {
            uint32_t v[LDC];
            if (LDC == 32) tmem_ld32(lane_base + static_cast<uint32_t>(b * BN + cc), v);
            else tmem_ld16(lane_base + static_cast<uint32_t>(b * BN + cc), v);
            tmem_wait_ld();
            // the bias enters with the first chunk (keeps it off the tile-boundary epilogue);
            // pairs of columns in packed fp32x2 (same round-to-nearest results)
            if (!HF && first) {
  #pragma unroll
              for (int u = 0; u < LDC; ++u) acc[cc + u] = sbias[boff + tc.n0 + col0 + cc + u];
            }
  #pragma unroll
            for (int u = 0; u < LDC; u += 2) {
              if (HF)
                ffma2_acc(acc[cc + u], acc[cc + u + 1], __uint_as_float(v[u]), __uint_as_float(v[u + 1]), f);
              else
                fadd2_acc(acc[cc + u], acc[cc + u + 1], __uint_as_float(v[u]), __uint_as_float(v[u + 1]));
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && c < 256 && warp == EP0 && lane == 0) g_tc_trace[10 * 256 + c] = clk();
          ++c;
          if (CH && kb == nk - 1) {
            // the first conv's tile is complete: h = act2(act1(acc)) split hi / lo exactly like
            // the transform would split it after a round trip through HBM (bit-identical to the
            // two-launch form), into the chained GEMM's A slots — this half's 64 columns are its
            // K-slabs 2 half and 2 half + 1
            const float s1 = slope_of(p.mid_act1, p.mid_alpha1), s2 = slope_of(p.mid_act2, p.mid_alpha2);
  #pragma unroll
            for (int j = 0; j < COLS / 32; ++j) {
              const int u = tcount * NK2 + half * (COLS / 32) + j, sl = u % NS2;
              const int pa = tcount * (nk + NK2) + nk + half * (COLS / 32) + j;  // A-ring position (SHR)
              if (SHR) mbar_wait(&aempty[pa % TS], ((pa / TS) + 1) & 1);  // MMAs of position pa - TS done
              else if (u >= NS2) mbar_wait(&a2empty[sl], ((u / NS2) + 1) & 1);  // MMAs of use u - NS2 done
              tc_fence_after();
              const uint32_t ta = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                  (SHR ? A_COL + 64 * (pa % TS) : A2_COL + W2 * sl);
              if (BF) {
                // the two-launch form rounds h to bf16 once in the first conv's epilogue when the
                // intermediate buffer holds bf16 (p.mid_bf), then applies act2 and rounds again
                uint32_t pk[16];
  #pragma unroll
                for (int e = 0; e < 16; ++e) {
                  float v0 = act_lin(acc[32 * j + 2 * e], s1), v1 = act_lin(acc[32 * j + 2 * e + 1], s1);
                  if (p.mid_bf) {
                    v0 = __bfloat162float(__float2bfloat16_rn(v0));
                    v1 = __bfloat162float(__float2bfloat16_rn(v1));
                  }
                  __nv_bfloat162 b2 = __floats2bfloat162_rn(act_lin(v0, s2), act_lin(v1, s2));
                  pk[e] = *reinterpret_cast<uint32_t*>(&b2);
                }
                tmem_st16(ta, pk);
              }
  #pragma unroll
              for (int h16 = 0; h16 < (BF ? 0 : 2); ++h16) {
                uint32_t hv[16], lv[16];
  #pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const float a = act_lin(act_lin(acc[32 * j + 16 * h16 + e], s1), s2);
                  const float hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
                  hv[e] = __float_as_uint(hi);
                  lv[e] = __float_as_uint(a - hi);
                }
                tmem_st16(ta + 16 * h16, hv);
                tmem_st16(ta + 32 + 16 * h16, lv);
              }
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&a2full[sl]);
            }
          }
        }
        // ---- epilogue: bias/act/gate (+ residual from staging) -> staging (TMA-stored by w14)
        const bool trace = (TC_DBG(p) & 32) && blockIdx.x == 0 && tcount < 64 && warp == EP0 && lane == 0;
        if (trace) g_tc_trace[6 * 256 + 4 * tcount + 0] = clk();
        if (p.res) {
          mbar_wait(res_full, tcount & 1);
        } else if (tcount > 0) {
          mbar_wait(stg_free, (tcount - 1) & 1);
        }
        if (trace) g_tc_trace[6 * 256 + 4 * tcount + 1] = clk();
        __nv_bfloat16* stgb = reinterpret_cast<__nv_bfloat16*>(stg);  // bf16 buffers (bf16 plans)
        if (p.gate) {
  #pragma unroll
          for (int u = 0; u < COLS; u += 2) {
            const float o = gate_fast(acc[u], acc[u + 1]);
            if (OBF)
              stgb[stg_off_b(r, (col0 + u) >> 1)] = __float2bfloat16_rn(o);
            else
              stg[stg_off(r, (col0 + u) >> 1)] = o;
          }
        } else if (OBF && p.post_act != ACT_TANH && p.res_act != ACT_TANH) {
          // bf16 output (and bf16 residual: a plan never mixes the two on one op), 4 columns per access
          const float ps = slope_of(p.post_act, p.post_alpha);
          const float rs = slope_of(p.res_act, p.res_alpha);
          const bool pmax = ps <= 1.f, rmax = rs <= 1.f, rid = rs == 1.f;
          auto lin = [](float v, float sl, bool mx) { return mx ? fmaxf(v, v * sl) : fminf(v, v * sl); };
  #pragma unroll
          for (int u = 0; u < COLS; u += 4) {
            uint2* dst = reinterpret_cast<uint2*>(stgb + stg_off_b(r, col0 + u));
            float o[4] = {lin(acc[u], ps, pmax), lin(acc[u + 1], ps, pmax), lin(acc[u + 2], ps, pmax),
                          lin(acc[u + 3], ps, pmax)};
            if (p.res) {
              const uint2 rv = *dst;
              const float2 r0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rv.x));
              const float2 r1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rv.y));
              const float rr[4] = {r0.x, r0.y, r1.x, r1.y};
  #pragma unroll
              for (int k = 0; k < 4; ++k) o[k] += rid ? rr[k] : lin(rr[k], rs, rmax);
            }
            __nv_bfloat162 a2 = __floats2bfloat162_rn(o[0], o[1]), b2 = __floats2bfloat162_rn(o[2], o[3]);
            uint2 w;
            w.x = *reinterpret_cast<uint32_t*>(&a2);
            w.y = *reinterpret_cast<uint32_t*>(&b2);
            *dst = w;
          }
        } else if (!OBF && p.post_act == ACT_ID && (!p.res || p.res_act == ACT_ID)) {
          // no activation on either operand (the residual units' convs): out = acc (+ skip),
          // packed fp32x2 adds
          // (skip rows read four vectors at a time ahead of their adds: one exposed
          // shared-memory latency per batch instead of one per vector)
          const bool has_res = p.res != nullptr;
          constexpr int EB = COLS >= 16 ? 16 : COLS;
  #pragma unroll
          for (int u0 = 0; u0 < COLS; u0 += EB) {
            float4 rv[EB / 4];
            if (has_res) {
  #pragma unroll
              for (int k = 0; k < EB / 4; ++k) rv[k] = *reinterpret_cast<const float4*>(stg + stg_off(r, col0 + u0 + 4 * k));
  #pragma unroll
              for (int k = 0; k < EB / 4; ++k) {
                const int u = u0 + 4 * k;
                fadd2_acc(acc[u], acc[u + 1], rv[k].x, rv[k].y);
                fadd2_acc(acc[u + 2], acc[u + 3], rv[k].z, rv[k].w);
              }
            }
  #pragma unroll
            for (int k = 0; k < EB / 4; ++k) {
              const int u = u0 + 4 * k;
              *reinterpret_cast<float4*>(stg + stg_off(r, col0 + u)) = make_float4(acc[u], acc[u + 1], acc[u + 2], acc[u + 3]);
            }
          }
        } else if (p.post_act != ACT_TANH && p.res_act != ACT_TANH) {
          // LeakyReLU(v) = max(v, a v) for a <= 1 (min for a > 1): 2 instructions
          const float ps = slope_of(p.post_act, p.post_alpha);
          const float rs = slope_of(p.res_act, p.res_alpha);
          const bool pmax = ps <= 1.f, rmax = rs <= 1.f, rid = rs == 1.f;
          auto lin = [](float v, float sl, bool mx) { return mx ? fmaxf(v, v * sl) : fminf(v, v * sl); };
  #pragma unroll
          for (int u = 0; u < COLS; u += 4) {
            float4* dst = reinterpret_cast<float4*>(stg + stg_off(r, col0 + u));
            float4 o;
            o.x = lin(acc[u], ps, pmax);
            o.y = lin(acc[u + 1], ps, pmax);
            o.z = lin(acc[u + 2], ps, pmax);
            o.w = lin(acc[u + 3], ps, pmax);
            if (p.res) {
              float4 rv = *dst;
              if (!rid) rv = make_float4(lin(rv.x, rs, rmax), lin(rv.y, rs, rmax), lin(rv.z, rs, rmax), lin(rv.w, rs, rmax));
              o.x += rv.x;
              o.y += rv.y;
              o.z += rv.z;
              o.w += rv.w;
            }
            *dst = o;
          }
        } else {  // tanh epilogues (unused by the five configs): out-of-line math
  #pragma unroll
          for (int u = 0; u < COLS; ++u) {
            const int n = tc.n0 + col0 + u;
            float o = act_apply(acc[u], p.post_act, p.post_alpha);
            if (OBF) {
              __nv_bfloat16* dst = stgb + stg_off_b(r, col0 + u);
              if (p.res) o += act_apply(__bfloat162float(*dst), p.res_act, p.res_alpha);
              *dst = __float2bfloat16_rn(o);
            } else {
              float* dst = stg + stg_off(r, col0 + u);
              if (p.res) o += act_apply(*dst, p.res_act, p.res_alpha);
              *dst = o;
            }
          }
        }
        if (trace) g_tc_trace[6 * 256 + 4 * tcount + 2] = clk();
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(stg_written);
        if (trace) g_tc_trace[6 * 256 + 4 * tcount + 3] = clk();
      }
  };
  auto role_win_prod = [&]() {
      // ===================== TMA producer, window mode =====================
      // per 32-channel block: the 128 + halo input rows once (window slot), then per tap the
      // weight hi / lo tiles into the W ring
      const int taps = nk / p.cblocks;
      const uint32_t a_bytes = static_cast<uint32_t>(BK * (ABF ? 2 : 4) * (p.R + p.halo));
      if (p.wres) {  // whole weight resident: slab kb = cb * taps + q at slot kb
        mbar_expect_tx_w(wres_full, static_cast<uint32_t>(nk) * 2 * L::B_TILE);
        for (int cb = 0; cb < p.cblocks; ++cb)
          for (int q = 0; q < taps; ++q) {
            const int kb = cb * taps + q, kw = (q * p.cblocks + cb) * BK;
            tma_load_3d_w(&tmap_w, wres_full, b_hi(kb), kw, 0, 0);
            tma_load_3d_w(&tmap_w, wres_full, b_lo(kb), kw, 0, 1);
          }
      }
      int g = 0, u = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
        for (int cb = 0; cb < p.cblocks; ++cb, ++u) {
          const int sa = u % L::AST;
          if (u >= L::AST) mbar_wait_bo<SC_SLEEP_PROD>(&wa_empty[sa], ((u / L::AST) + 1) & 1);
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && u < 256 && lane == 0) g_tc_trace[0 * 256 + u] = clk();
          mbar_expect_tx_w(&wa_full[sa], a_bytes);
          tma_load_3d_w(&tmap_a, &wa_full[sa], win_hi(sa), p.a_c0 + cb * BK, p.a_row0 + tc.i0, tc.s0);
          // warm L2 with the next tile's window of this channel block: two fp32 window slots
          // cannot cover the DRAM latency of the next load on their own (bf16 tiles hold three
          // slots; there the prefetch cost 15-25% on cfg3's strided / ConvT layers)
          if (!BF && tile + static_cast<int>(gridDim.x) < n_tiles && lane == 0) {
            const TileCoord tn = tile_coord(p, tile + gridDim.x, n_tiles_n, BN);
            tma_prefetch_3d(&tmap_a, p.a_c0 + cb * BK, p.a_row0 + tn.i0, tn.s0);
          }
          if (p.wres) continue;
          for (int q = 0; q < taps; ++q, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait_bo<SC_SLEEP_PROD>(&empty[s], ((g / STAGES) + 1) & 1);
            const int kw = (q * p.cblocks + cb) * BK;
            mbar_expect_tx_w(&full[s], (BF ? 1 : 2) * L::B_TILE);
            tma_load_3d_w(&tmap_w, &full[s], b_hi(s), kw, tc.n0, 0);
            if (!BF) tma_load_3d_w(&tmap_w, &full[s], b_lo(s), kw, tc.n0, 1);
          }
        }
        for (int k2 = 0; k2 < NK2; ++k2, ++g) {  // chained conv's weight slabs (bf16)
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait_bo<SC_SLEEP_PROD>(&empty[s], ((g / STAGES) + 1) & 1);
          mbar_expect_tx_w(&full[s], L::B_TILE);
          tma_load_3d_w(&tmap_w, &full[s], b_hi(s), (nk + k2) * BK, tc.n0, 0);
        }
      }
  };
  auto role_win_mma = [&]() {
      // ===================== MMA issuer, window mode (SS-MMAs at a per-tap row offset) ========
      const uint32_t tbase = warp_uniform(tmem_base);
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(BM >> 4) << 24);
      const int taps = nk / p.cblocks;
      int g = 0, c = 0, tcount = 0, u = 0;
      if (p.wres) mbar_wait(wres_full, 0);
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        for (int cb = 0; cb < p.cblocks; ++cb, ++u) {
          const int sa = u % L::AST;
          mbar_wait(&wa_ready[sa], (u / L::AST) & 1);
          tc_fence_after();
          const uint32_t wh = smem_u32(win_hi(sa)), wl = smem_u32(win_lo(sa));
          const uint64_t wdesc_h = sw64_desc(wh);  // 3xFP16: this window's fp16 hi plane
          for (int q = 0; q < taps; ++q, ++g) {
            const int kb = cb * taps + q;
            const int s = g % STAGES;
            const int b = c % NB;
            const bool chunk_first = (kb % CK) == 0;
            const bool chunk_last = ((kb % CK) == CK - 1) || (kb == nk - 1);
            if (chunk_first && c >= NB) mbar_wait(&tempty[b], ((c / NB) + 1) & 1);
            if (!p.wres) mbar_wait(&full[s], (g / STAGES) & 1);
            tc_fence_after();
            const uint32_t dmain = tbase + static_cast<uint32_t>(b * BN);
            if (BF) {  // one bf16 window copy, SW64 rows of 64 B: tap q starts q * tap_rows rows in
              const uint32_t idesc_bf = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                        (static_cast<uint32_t>(BM >> 4) << 24);
              const uint32_t offb = static_cast<uint32_t>(q * p.a_tap_rows * BK * 2);
              const uint32_t wb = smem_u32(win_bf(sa)), bb = smem_u32(b_hi(s));
  #pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t acc0 = (!chunk_first || kk > 0) ? 1u : 0u;
                mma_bf16_w(dmain, sw64_desc(wb + offb + kk * 32), sw64_desc(bb + kk * 32), idesc_bf, acc0);
              }
            } else if (HF) {  // fp16 hi / lo window planes (SW64 rows of 64 B), tap q at a row offset
              const uint32_t idesc_h = (1u << 4) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                       (static_cast<uint32_t>(BM >> 4) << 24);  // F32 += F16 x F16
              // descriptors by addition: the window's hi plane + the tap's row offset (64 B rows:
              // 4 address units per row); lo plane / W lo tile at fixed distances
              const int ws = p.wres ? kb : s;
              const uint64_t ah = wdesc_h + static_cast<uint64_t>(q * p.a_tap_rows * 4);
              const uint64_t bh = sw64_desc(smem_u32(b_hi(ws)));
              mma_f16x3_slab_ss_w(dmain, ah, ah + (L::WROWS * BK * 2) / 16, bh, bh + L::B_TILE / 16, idesc_h,
                                  chunk_first ? 0u : 1u);
            } else {
              const uint32_t off = static_cast<uint32_t>(q * p.a_tap_rows * BK * 4);
              const int ws = p.wres ? kb : s;
              if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[3 * 256 + g] = clk();
              const uint32_t bh = smem_u32(b_hi(ws)), bl = smem_u32(b_lo(ws));
              // corrections first (2^-10 of the signal), then the main product, all into this
              // chunk's accumulator: the truncating accumulation meets the large terms only in
              // its last four steps (same error as a separate correction accumulator)
  #pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {
                const uint32_t acc0 = (!chunk_first || kk > 0) ? 1u : 0u;
                mma_tf32_w(dmain, sw128_desc(wl + off + kk * 32), sw128_desc(bh + kk * 32), idesc, acc0);
                mma_tf32_w(dmain, sw128_desc(wh + off + kk * 32), sw128_desc(bl + kk * 32), idesc, 1u);
              }
  #pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk)
                mma_tf32_w(dmain, sw128_desc(wh + off + kk * 32), sw128_desc(bh + kk * 32), idesc, 1u);
            }
            if (!p.wres) mma_commit_w(&empty[s]);
            if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[11 * 256 + g] = clk();
            if (chunk_last) {
              mma_commit_w(&tfull[b]);
              ++c;
            }
          }
          mma_commit_w(&wa_empty[sa]);
        }
        if (CH) {  // chained 1x1 GEMM (bf16): A from the drain's TMEM slots, one chunk accumulator
          const uint32_t idesc_bf = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(BM >> 4) << 24);
          for (int k2 = 0; k2 < NK2; ++k2, ++g) {
            const int s = g % STAGES;
            const int b = c % NB;
            const int u2 = tcount * NK2 + k2, sl = u2 % NS2;
            if (k2 == 0 && c >= NB) mbar_wait(&tempty[b], ((c / NB) + 1) & 1);
            mbar_wait(&full[s], (g / STAGES) & 1);
            mbar_wait(&a2full[sl], (u2 / NS2) & 1);
            tc_fence_after();
            const uint32_t dmain = tbase + static_cast<uint32_t>(b * BN);
            const uint32_t bb = smem_u32(b_hi(s)), at = tbase + A2_COL + W2 * sl;
  #pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_bf16_ts_w(dmain, at + kk * 8, sw64_desc(bb + kk * 32), idesc_bf, (k2 > 0 || kk > 0) ? 1u : 0u);
            mma_commit_w(&a2empty[sl]);
            mma_commit_w(&empty[s]);
            if (k2 == NK2 - 1) {
              mma_commit_w(&tfull[b]);
              ++c;
            }
          }
        }
      }
  };
  auto role_win_xf = [&]() {
      // ===================== transform, window mode: hi in place, lo to the lo window ==========
      // (3xFP16: two sets of four warps take alternate windows, each with its own named barrier)
      const int xset = RX ? (warp - Roles<RX>::XF0) >> 2 : 0;
      const int t = threadIdx.x - (Roles<RX>::XF0 + 4 * xset) * 32;  // 0..127
      const bool pre_tanh = p.pre_act == ACT_TANH;
      const float pre_s = slope_of(p.pre_act, p.pre_alpha);
      const int rows = p.R + p.halo;
      int u = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int cb = 0; cb < p.cblocks; ++cb, ++u) {
          if (RX && (u & 1) != xset) continue;
          const int sa = u % L::AST;
          mbar_wait_bo<SC_SLEEP_XF>(&wa_full[sa], (u / L::AST) & 1);
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && u < 256 && t == 0) g_tc_trace[1 * 256 + u] = clk();
          if (BF) {
            // raw fp32 rows (SW128, 16B chunk j at j ^ (w & 7)) -> pre-activation -> bf16 copy
            // (SW64 rows of 64 B, 16B chunk jo at jo ^ ((w >> 1) & 3)); item = (row, output chunk)
            uint4* bfr = reinterpret_cast<uint4*>(win_bf(sa));
            if (ABF) {  // the window rows are bf16 already (SW64): pre-activation into the copy
              const uint4* rawb = reinterpret_cast<const uint4*>(win_hi(sa));
              for (int e = t; e < rows * 4; e += 128) {
                const int w = e >> 2, jp = (e & 3) ^ ((w >> 1) & 3);
                uint4 u = rawb[w * 4 + jp];
                if (pre_tanh || pre_s != 1.f) {
                  uint32_t wv[4] = {u.x, u.y, u.z, u.w};
  #pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    if (!pre_tanh && pre_s < 1.f) {  // exact LeakyReLU on the packed pair
                      const float lo = __uint_as_float(wv[k] << 16), hi = __uint_as_float(wv[k] & 0xFFFF0000u);
                      __nv_bfloat162 b2 = __floats2bfloat162_rn(fmaxf(lo, lo * pre_s), fmaxf(hi, hi * pre_s));
                      wv[k] = *reinterpret_cast<uint32_t*>(&b2);
                    } else {
                      float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[k]));
                      f.x = pre_tanh ? tanh_ool(f.x) : act_lin(f.x, pre_s);
                      f.y = pre_tanh ? tanh_ool(f.y) : act_lin(f.y, pre_s);
                      __nv_bfloat162 b2 = __floats2bfloat162_rn(f.x, f.y);
                      wv[k] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                  }
                  u = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
                bfr[w * 4 + jp] = u;
              }
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) mbar_arrive(&wa_ready[sa]);
              continue;
            }
            const float4* raw = reinterpret_cast<const float4*>(win_hi(sa));
            constexpr int IPB = (L::WROWS * 4 + 127) / 128;
            float4 v[IPB][2];
  #pragma unroll
            for (int i = 0; i < IPB; ++i) {
              const int e = t + 128 * i, w = e >> 2, jo = e & 3;
              if (w < rows) {
                v[i][0] = raw[w * 8 + ((2 * jo) ^ (w & 7))];
                v[i][1] = raw[w * 8 + ((2 * jo + 1) ^ (w & 7))];
              }
            }
  #pragma unroll
            for (int i = 0; i < IPB; ++i) {
              const int e = t + 128 * i, w = e >> 2, jo = e & 3;
              if (w >= rows) continue;
              float x[8] = {v[i][0].x, v[i][0].y, v[i][0].z, v[i][0].w, v[i][1].x, v[i][1].y, v[i][1].z, v[i][1].w};
              uint32_t pk[4];
  #pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float y0 = pre_tanh ? tanh_ool(x[2 * k]) : act_lin(x[2 * k], pre_s);
                const float y1 = pre_tanh ? tanh_ool(x[2 * k + 1]) : act_lin(x[2 * k + 1], pre_s);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(y0, y1);
                pk[k] = *reinterpret_cast<uint32_t*>(&b2);
              }
              bfr[w * 4 + (jo ^ ((w >> 1) & 3))] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&wa_ready[sa]);
            continue;
          }
          if (HF) {
            // raw fp32 rows (SW128, 16B chunk j of row w at j ^ (w & 7)) -> pre-activation ->
            // per-row power-of-two scale -> fp16 hi | lo planes written IN PLACE over the raw rows
            // (SW64 rows of 64 B: 16B chunk jb of row w at jb ^ ((w >> 1) & 3)), once every
            // thread of the four warps has read its rows (named barrier 1).  Thread t owns row t
            // whole (no shuffles) plus one 16-byte item of the halo rows 128 .. 143 (8 lanes per
            // row, max by three shuffles).  Rows past the window are converted too (stale data,
            // never read by an MMA): no branches, so the two rows' math interleaves.
            const float4* raw = reinterpret_cast<const float4*>(win_hi(sa));
            float4 v[8];
  #pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = raw[t * 8 + (j ^ (t & 7))];
            const int we = BM + (t >> 3), je = t & 7;
            const float4 ve = raw[we * 8 + (je ^ (we & 7))];
            named_bar(1 + xset, 128);
            uint8_t* rsw = rsc + (u % RS_WIN) * L::WROWS;
            const int s_lo = -126 > -127 - p.f16_sw ? -126 : -127 - p.f16_sw;
            const int s_hi = 127 < 126 - p.f16_sw ? 127 : 126 - p.f16_sw;
            {
              float m = 0.f;
  #pragma unroll
              for (int j = 0; j < 8; ++j)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
              int sx = 14 - (static_cast<int>(__float_as_uint(m) >> 23) - 127);
              sx = sx < s_lo ? s_lo : sx > s_hi ? s_hi : sx;
              const float sc = __uint_as_float(static_cast<uint32_t>(127 + sx) << 23);
              const float scn = sc * pre_s;
              uint32_t hv[16], lv[16];
  #pragma unroll
              for (int k = 0; k < 16; ++k) {
                const float x0 = (k & 1) ? v[k >> 1].z : v[k >> 1].x, x1 = (k & 1) ? v[k >> 1].w : v[k >> 1].y;
                // identity / LeakyReLU with |slope| <= 1 only (plan time: tanh and larger slopes
                // keep the layer on 3xTF32)
                const float2 p2 = fmul2s(x0, x1, sc), n2 = fmul2s(x0, x1, scn);
                const float2 t2 = make_float2(fmaxf(p2.x, n2.x), fmaxf(p2.y, n2.y));
                split_f16x2(t2, hv[k], lv[k]);
              }
              uint4* hr = reinterpret_cast<uint4*>(win_hi(sa)) + t * 4;
              uint4* lr = reinterpret_cast<uint4*>(win_lo16(sa)) + t * 4;
  #pragma unroll
              for (int jb = 0; jb < 4; ++jb) {
                hr[jb ^ ((t >> 1) & 3)] = make_uint4(hv[4 * jb], hv[4 * jb + 1], hv[4 * jb + 2], hv[4 * jb + 3]);
                lr[jb ^ ((t >> 1) & 3)] = make_uint4(lv[4 * jb], lv[4 * jb + 1], lv[4 * jb + 2], lv[4 * jb + 3]);
              }
              rsw[t] = static_cast<uint8_t>(127 - sx - p.f16_sw);
            }
            {
              float m = fmaxf(fmaxf(fabsf(ve.x), fabsf(ve.y)), fmaxf(fabsf(ve.z), fabsf(ve.w)));
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
              int sx = 14 - (static_cast<int>(__float_as_uint(m) >> 23) - 127);
              sx = sx < s_lo ? s_lo : sx > s_hi ? s_hi : sx;
              const float sc = __uint_as_float(static_cast<uint32_t>(127 + sx) << 23);
              const float scn = sc * pre_s;
              uint32_t hv[2], lv[2];
  #pragma unroll
              for (int k = 0; k < 2; ++k) {
                const float x0 = k ? ve.z : ve.x, x1 = k ? ve.w : ve.y;
                // identity / LeakyReLU with |slope| <= 1 only (plan time: tanh and larger slopes
                // keep the layer on 3xTF32)
                const float2 p2 = fmul2s(x0, x1, sc), n2 = fmul2s(x0, x1, scn);
                const float2 t2 = make_float2(fmaxf(p2.x, n2.x), fmaxf(p2.y, n2.y));
                split_f16x2(t2, hv[k], lv[k]);
              }
              const int po = we * 8 + (((je >> 1) ^ ((we >> 1) & 3)) << 1) + (je & 1);  // uint2 units
              reinterpret_cast<uint2*>(win_hi(sa))[po] = make_uint2(hv[0], hv[1]);
              reinterpret_cast<uint2*>(win_lo16(sa))[po] = make_uint2(lv[0], lv[1]);
              if (je == 0) rsw[we] = static_cast<uint8_t>(127 - sx - p.f16_sw);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&wa_ready[sa]);
            continue;
          }
          float4* hrow = reinterpret_cast<float4*>(win_hi(sa));
          float4* lrow = reinterpret_cast<float4*>(win_lo(sa));
          // (row, 16B chunk) items spread evenly over the 128 threads, all loads issued first;
          // 8 consecutive items = the 8 chunks of one row: conflict-free 128-bit accesses
          constexpr int IPT = (WIN_ROWS * 8 + 127) / 128;  // items per thread (9)
          float4 v[IPT];
  #pragma unroll
          for (int i = 0; i < IPT; ++i) {
            const int e = t + 128 * i, w = e >> 3;
            if (w < rows) v[i] = hrow[w * 8 + ((e & 7) ^ (w & 7))];
          }
  #pragma unroll
          for (int i = 0; i < IPT; ++i) {
            const int e = t + 128 * i, w = e >> 3;
            if (w >= rows) continue;
            const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
            float h[4], l[4];
  #pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float y = pre_tanh ? tanh_ool(x[k]) : act_lin(x[k], pre_s);
              h[k] = __uint_as_float(__float_as_uint(y) & 0xFFFFE000u);
              l[k] = y - h[k];
            }
            const int pj = w * 8 + ((e & 7) ^ (w & 7));
            hrow[pj] = make_float4(h[0], h[1], h[2], h[3]);
            lrow[pj] = make_float4(l[0], l[1], l[2], l[3]);
          }
          fence_proxy_async();  // generic smem writes -> read by the tensor core (async proxy)
          __syncwarp();
          if (lane == 0) mbar_arrive(&wa_ready[sa]);
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && u < 256 && t == 0) g_tc_trace[2 * 256 + u] = clk();
        }
      }
  };
  if constexpr (RX) {
    // 3xFP16: warpgroup-aligned roles with register reallocation (setmaxnreg): WG0 = W / window
    // producer, MMA issuer, epilogue I/O, A-unit producer (X2) (48 registers); WG1-2 = the two
    // transform sets, alternate K-slabs (X2) or windows (88); WG3-4 = drain + epilogue (128: a
    // 64-column fp32 accumulator per thread)
    if (warp < 4) {
      reg_dealloc<48>();
      if (WIN && warp == 0) {
        role_win_prod();
      } else if (WIN && warp == 1) {
        role_win_mma();
      } else if (WIN && warp == 3) {
        // (no A-unit producer in window mode)
      } else if (warp == 0) {
        // ===================== W producer, X2: weight hi | lo tiles into the stage ring ==========
        const int taps = nk / p.cblocks;
        int g = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
          const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
          int cb = 0, q = 0;
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int s = g % STAGES;
            if (g >= STAGES) mbar_wait_bo<SC_SLEEP_PROD>(&empty[s], ((g / STAGES) + 1) & 1);
            if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[0 * 256 + g] = clk();
            const int kw = (q * p.cblocks + cb) * BK;
            mbar_expect_tx_w(&full[s], 2 * L::B_TILE);
            tma_load_3d_w(&tmap_w, &full[s], b_hi(s), kw, tc.n0, 0);
            tma_load_3d_w(&tmap_w, &full[s], b_lo(s), kw, tc.n0, 1);
            if (p.cbmaj) {
              if (++q == taps) q = 0, ++cb;
            } else if (++cb == p.cblocks) {
              cb = 0, ++q;
            }
          }
        }
      } else if (warp == 1) {
        role_mma();
      } else if (warp == IO_WARP) {
        role_io();
      } else {
        // ===================== A-unit producer, X2 =====================
        // A unit = the rows of one K-slab (p.awin = 0), or of one 32-channel block for every tap:
        // G streams x (R + halo) rows (p.awin = 1: the taps' boxes overlap, so one load serves them).
        // Limited only by the unit ring (released by the transform), not by the W ring.
        const int taps = nk / p.cblocks;
        const uint32_t abytes = static_cast<uint32_t>(BK * 4 * (p.R + (p.awin ? p.halo : 0)) * p.G);
        int u = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
          const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
          int cb = 0, q = 0;
          for (int kb = 0; kb < nk; ++kb) {
            if (!p.awin || q == 0) {
              // awin: three window slots in turn (every transform warp reads every unit);
              // per-slab units: four 16 KB slots, two private to each transform set (slabs
              // alternate between the sets, and a set only watches its own units' barriers)
              const int sa = p.awin ? u % L::AST : ((u & 1) << 1) | ((u >> 1) & 1);
              const int use = p.awin ? u / L::AST : u >> 2;
              if (use > 0) mbar_wait_bo<SC_SLEEP_PROD>(&wa_empty[sa], (use + 1) & 1);
              mbar_expect_tx_w(&wa_full[sa], abytes);
              tma_load_3d_w(&tmap_a, &wa_full[sa], p.awin ? win_hi(sa) : wins + sa * A_TILE, p.a_c0 + cb * BK,
                            p.a_row0 + tc.i0 + (p.awin ? 0 : q * p.a_tap_rows), tc.s0);
              ++u;
            }
            if (p.cbmaj) {
              if (++q == taps) q = 0, ++cb;
            } else if (++cb == p.cblocks) {
              cb = 0, ++q;
            }
          }
        }
      }
    } else if (warp < Roles<RX>::EP0) {
      reg_dealloc<88>();
      if (WIN) {
        role_win_xf();
      } else {
      // ===================== transform, X2 (w3..w10: two sets of four, alternate K-slabs) =====
      // thread = tile row r (= TMEM lane): the row's power-of-two scale, pre-activation folded
      // into the scaling (LeakyReLU(x) 2^s = max(x 2^s, x (a 2^s)) exactly: 2^s is a power of
      // two), fp16 hi | lo pairs (low half = even k) into this slab's TMEM A slot; the unscale
      // exponent of (row, slab) goes to the ring the drain reads.  The scale is taken from
      // max |x| (>= max |act(x)|: LeakyReLU slopes are <= 1 here, plan time; tanh: <= |x|) — the same rule as the window
      // transform, so both modes produce identical operands.  Tile row r = (stream r / R, frame
      // r % R); its input row sits at r in a per-slab unit, or at (r / R)(R + halo) + r % R + q
      // tap_rows in a block window (p.awin).  A transform warp releases a unit after its own last
      // read of it (having seen it land: a release can never run ahead into the slot's previous use).
      const int xset = (warp - Roles<X2>::XF0) >> 2;
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const int taps = nk / p.cblocks;
      // rows past G x R (a partial tile) are never stored: read any in-slot row for them
      const int srow = (!p.awin || r >= p.G * p.R) ? (r < p.G * p.R ? r : 0) : (r / p.R) * (p.R + p.halo) + r % p.R;
      const float pre_s = slope_of(p.pre_act, p.pre_alpha);
      const int s_lo = -126 > -127 - p.f16_sw ? -126 : -127 - p.f16_sw;
      const int s_hi = 127 < 126 - p.f16_sw ? 127 : 126 - p.f16_sw;
      // Each set walks only its own slabs (g = xset, xset + 2, ...; g counts across tiles).  The
      // tail of a slab — TMEM store completion, fence, arrive — is deferred into the next own
      // slab, after that slab's loads have been issued, and the A-slot wait is taken there too
      // (it has long completed): both latencies overlap the shared-memory loads instead of
      // idling the warp (per-quarter traces: ~300 of ~1950 cycles per slab pair).  A warp
      // releases a unit right after its own last read of it (awin: both sets read every unit, 8
      // arrivals; per-slab units: the handling set's 4).
      int g = xset, kb = xset, tile = blockIdx.x, tcount = 0;
      while (tile < n_tiles && kb >= nk) kb -= nk, tile += gridDim.x, ++tcount;
      int cb = p.awin ? kb / taps : 0, q = p.awin ? kb % taps : 0;
      int prev_s = -1;
      const uint32_t tq = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + A_COL;
      while (tile < n_tiles) {
        const int u = p.awin ? tcount * p.cblocks + cb : g;
        const bool last_read = !p.awin || q + 2 >= taps;
        const int sa = p.awin ? u % L::AST : ((u & 1) << 1) | ((u >> 1) & 1);  // see the A-unit producer
        mbar_wait_bo<SC_SLEEP_XF>(&wa_full[sa], (p.awin ? u / L::AST : u >> 2) & 1);
        const bool trq = (TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0;  // rows 16 + 4 quarter ..
        if (trq) g_tc_trace[(16 + 4 * quarter) * 256 + g] = clk();
        const int wr = srow + (p.awin ? q * p.a_tap_rows : 0);
        const float4* row = reinterpret_cast<const float4*>(p.awin ? win_hi(sa) : wins + sa * A_TILE) + wr * 8;
        float4 v[8];
  #pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = row[j ^ (wr & 7)];
        // while the loads are in flight: this slab's A slot (MMAs of g - TS done), then the
        // previous own slab's deferred tail
        if (g >= TS) mbar_wait(&aempty[g % TS], ((g / TS) + 1) & 1);
        if (prev_s >= 0) {
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xform[prev_s]);
        }
        tc_fence_after();
        float m = 0.f;
  #pragma unroll
        for (int j = 0; j < 8; ++j)
          m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
        // this warp's reads of the unit are done once m (a function of every loaded value)
        // exists: release the slot only then — an arrive right after the LDS instructions
        // could let the next TMA fill overwrite rows still in flight to the registers
        if (last_read) {
          m = __shfl_sync(0xffffffffu, m, lane);  // consume m before the arrive
          __syncwarp();
          if (lane == 0) mbar_arrive(&wa_empty[sa]);
        }
        int sx = 14 - (static_cast<int>(__float_as_uint(m) >> 23) - 127);
        sx = sx < s_lo ? s_lo : sx > s_hi ? s_hi : sx;
        const float sc = __uint_as_float(static_cast<uint32_t>(127 + sx) << 23);
        const float scn = sc * pre_s;  // exact
        uint32_t hv[16], lv[16];
  #pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float x0 = (k & 1) ? v[k >> 1].z : v[k >> 1].x, x1 = (k & 1) ? v[k >> 1].w : v[k >> 1].y;
          // identity / LeakyReLU with |slope| <= 1 only (plan time: tanh and larger slopes keep
          // the layer on 3xTF32)
          const float2 p2 = fmul2s(x0, x1, sc), n2 = fmul2s(x0, x1, scn);
          const float2 t2 = make_float2(fmaxf(p2.x, n2.x), fmaxf(p2.y, n2.y));
          split_f16x2(t2, hv[k], lv[k]);
        }
        rsc[(g % RS_RING) * BM + r] = static_cast<uint8_t>(127 - sx - p.f16_sw);
        if (trq) g_tc_trace[(17 + 4 * quarter) * 256 + g] = clk();
        const uint32_t ta = tq + 32 * (g % TS);
        tmem_st16(ta, hv);
        tmem_st16(ta + 16, lv);
        // no proxy fence: nothing was written to shared memory for the async proxy (the A
        // slot is TMEM; the unit is only read), and the scale byte is read by the drain
        prev_s = g % STAGES;
        if (trq) g_tc_trace[(18 + 4 * quarter) * 256 + g] = clk();
        g += 2, kb += 2;
        if (p.awin) {
          q += 2;
          if (q >= taps) q -= taps, ++cb;
        }
        if (kb >= nk) {
          do kb -= nk, tile += gridDim.x, ++tcount; while (kb >= nk);
          if (p.awin) cb = kb / taps, q = kb - cb * taps;
        }
      }
      if (prev_s >= 0) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xform[prev_s]);
      }
      }
    } else {
      reg_alloc<128>();
      role_drain();
    }
  } else if (WIN && warp == 0) {
    role_win_prod();
  } else if (WIN && warp == 1) {
    role_win_mma();
  } else if (WIN && warp >= XF_WARP0 && warp < EP0) {
    role_win_xf();
  } else if (warp == 0) {
    // ===================== TMA producer (whole warp, one elected lane issues) =====================
    {
      const uint32_t bytes = static_cast<uint32_t>(BK * (ABF ? 2 : 4) * p.R * p.G) + (BF ? 1 : 2) * L::B_TILE;
      int g = 0;
      const int taps = nk / p.cblocks;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
        int cb = 0, q = 0;  // this slab's 32-channel block and tap (advanced below, no divisions)
        for (int kb = 0; kb < nkt; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait_bo<SC_SLEEP_PROD>(&empty[s], ((g / STAGES) + 1) & 1);
          if (CH && kb >= nk) {  // chained conv's weight slab only (its A comes from the drain)
            if (BF) {
              mbar_expect_tx_w(&full[s], L::B_TILE);
              tma_load_3d_w(&tmap_w, &full[s], b_bf(s), kb * BK, tc.n0, 0);
            } else {
              mbar_expect_tx_w(&full[s], 2 * L::B_TILE);
              tma_load_3d_w(&tmap_w, &full[s], b_hi(s), kb * BK, tc.n0, 0);
              tma_load_3d_w(&tmap_w, &full[s], b_lo(s), kb * BK, tc.n0, 1);
            }
            continue;
          }
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[4 * 256 + g] = clk();
          // K-slab order: a layer that may also run in window mode (cbmaj) takes the window
          // mode's order (32-channel block major, tap minor), so its outputs do not depend on
          // the per-call tile geometry (bit-identical across buffer partitions);
          // the others take tap-major order (2% faster: the taps of one row block stay in L2)
          const int kw = (q * p.cblocks + cb) * BK;
          if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && lane == 0) g_tc_trace[0 * 256 + g] = clk();
          mbar_expect_tx_w(&full[s], bytes);
          tma_load_3d_w(&tmap_a, &full[s], a_hi(s), p.a_c0 + cb * BK, p.a_row0 + tc.i0 + q * p.a_tap_rows, tc.s0);
          if (BF) {
            tma_load_3d_w(&tmap_w, &full[s], b_bf(s), kw, tc.n0, 0);
          } else {
            tma_load_3d_w(&tmap_w, &full[s], b_hi(s), kw, tc.n0, 0);
            tma_load_3d_w(&tmap_w, &full[s], b_lo(s), kw, tc.n0, 1);
          }
          if (p.cbmaj) {
            if (++q == taps) q = 0, ++cb;
          } else if (++cb == p.cblocks) {
            cb = 0, ++q;
          }
        }
      }
    }
  } else if (warp == 1) {
    role_mma();
  } else if (warp == IO_WARP) {
    role_io();
  } else if (warp >= XF_WARP0 && warp < EP0) {
    // ===================== transform (w3..w6) =====================
    const int t = threadIdx.x - XF_WARP0 * 32;  // 0..127
    int g = 0, ga = 0;  // ga: A-ring slab counter (the chained conv's slabs skip the transform)
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < nkt; ++kb, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        if (CH && kb >= nk) {  // chained conv's weight slab: nothing to transform, but every
          __syncwarp();        // stage passes through here once per use (barrier phases)
          if (lane == 0) mbar_arrive(&xform[s]);
          continue;
        }
        if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && t == 0) g_tc_trace[1 * 256 + g] = clk();
        if (BF) {
          // thread = tile row r (= TMEM lane): fp32 SW128 row (16B chunk j at j ^ (r & 7)) ->
          // pre-activation -> bf16 pairs (low half = even k) -> this stage's TMEM A columns
          const int quarter = warp & 3;
          const int r = quarter * 32 + lane;
          const float4* row = reinterpret_cast<const float4*>(a_hi(s)) + r * 8;
          const bool pre_tanh = p.pre_act == ACT_TANH;
          const float pre_s = slope_of(p.pre_act, p.pre_alpha);
          uint32_t pk[16];
          if (ABF) {
            // bf16 buffer: SW64 row of 64 B (16B chunk jb at jb ^ ((r >> 1) & 3)), bf16 pairs
            const uint4* rowb = reinterpret_cast<const uint4*>(a_hi(s)) + r * 4;
            // LeakyReLU on a packed pair, exact: unpack by shifts, max(x, a x) in fp32 (a <= 1),
            // one round-to-nearest pack (the fp32 route's rounding) — 7 instructions per pair
            const bool ident = !pre_tanh && pre_s == 1.f;
            const bool pk_lrelu = !pre_tanh && pre_s < 1.f;
#pragma unroll
            for (int jb = 0; jb < 4; ++jb) {
              const uint4 u = rowb[jb ^ ((r >> 1) & 3)];
              const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (ident) {
                  pk[4 * jb + k] = w[k];
                } else if (pk_lrelu) {
                  const float lo = __uint_as_float(w[k] << 16), hi = __uint_as_float(w[k] & 0xFFFF0000u);
                  __nv_bfloat162 b2 = __floats2bfloat162_rn(fmaxf(lo, lo * pre_s), fmaxf(hi, hi * pre_s));
                  pk[4 * jb + k] = *reinterpret_cast<uint32_t*>(&b2);
                } else {
                  float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
                  f.x = pre_tanh ? tanh_ool(f.x) : act_lin(f.x, pre_s);
                  f.y = pre_tanh ? tanh_ool(f.y) : act_lin(f.y, pre_s);
                  __nv_bfloat162 b2 = __floats2bfloat162_rn(f.x, f.y);
                  pk[4 * jb + k] = *reinterpret_cast<uint32_t*>(&b2);
                }
              }
            }
          }
          if (!ABF) {
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 v = row[j4 ^ (r & 7)];
            if (pre_tanh) {
              v = make_float4(tanh_ool(v.x), tanh_ool(v.y), tanh_ool(v.z), tanh_ool(v.w));
            } else {
              v = make_float4(act_lin(v.x, pre_s), act_lin(v.y, pre_s), act_lin(v.z, pre_s), act_lin(v.w, pre_s));
            }
            __nv_bfloat162 lo2 = __floats2bfloat162_rn(v.x, v.y);
            __nv_bfloat162 hi2 = __floats2bfloat162_rn(v.z, v.w);
            pk[2 * j4] = *reinterpret_cast<uint32_t*>(&lo2);
            pk[2 * j4 + 1] = *reinterpret_cast<uint32_t*>(&hi2);
          }
          }
          const int a = ga % TS;
          if (ga >= TS) mbar_wait(&aempty[a], ((ga / TS) + 1) & 1);  // MMAs of ga - TS done
          tc_fence_after();
          tmem_st16(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + A_COL + 16 * a, pk);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
        }
        if (!BF) {
          // thread = tile row r (= TMEM lane): SW128 chunk j of row r lives at j ^ (r & 7); hi
          // and lo go to this stage's TMEM A columns (the MMAs read A from TMEM)
          const int quarter = warp & 3;
          const int r = quarter * 32 + lane;
          const float4* row = reinterpret_cast<const float4*>(a_hi(s)) + r * 8;
          const bool pre_tanh = p.pre_act == ACT_TANH;
          const float pre_s = slope_of(p.pre_act, p.pre_alpha);
          float hi[32], lo[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 v = row[j ^ (r & 7)];
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float a = pre_tanh ? tanh_ool(x[u]) : act_lin(x[u], pre_s);
              hi[4 * j + u] = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
              lo[4 * j + u] = a - hi[4 * j + u];
            }
          }
          const int a = ga % TS;
          if (ga >= TS) mbar_wait(&aempty[a], ((ga / TS) + 1) & 1);  // MMAs of ga - TS done
          tc_fence_after();
          const uint32_t ta = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + A_COL + 64 * a;
          tmem_st32(ta, hi);
          tmem_st32(ta + 32, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
        }
        ++ga;
        if (SHR && kb == nk - 1) ga += NK2;  // the chained slabs' ring positions (drain-written)
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xform[s]);
        if ((TC_DBG(p) & 32) && blockIdx.x == 0 && g < 256 && t == 0) g_tc_trace[2 * 256 + g] = clk();
      }
    }
  } else if (warp >= EP0) {
    role_drain();
  }

  tc_fence_before();
  __syncthreads();
  if ((TC_DBG(p) & 32) && threadIdx.x == 0 && blockIdx.x < 256) g_tc_trace[8 * 256 + blockIdx.x] = clk();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

// programmatic dependent launch of the tensor-core convs (SC_PDL=0 disables)
bool pdl_enabled() {
  static const int on = [] {
    const char* e = std::getenv("SC_PDL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on != 0;
}

// SM count per device ordinal (plans may live on different GPUs of one process)
std::atomic<int> g_num_sms[64];

int num_sms(int dev) {
  int n = g_num_sms[dev & 63].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

template <int BN, int STAGES, int CK, bool BF, bool WIN = false, int IOB = 0, bool CH = false, bool HF = false>
void launch_bn(const CUtensorMap& ma, const CUtensorMap& mw, const CUtensorMap& mo, const CUtensorMap& mr,
               const TcParams& p, cudaStream_t st) {
  using L = TcSmem<BN, STAGES, BF, WIN, IOB, HF>;
  static_assert(L::BYTES <= 232448, "shared memory budget");
  // cudaFuncSetAttribute applies to the CURRENT device only: track it per device ordinal.  A
  // concurrent first launch on two threads just sets the (idempotent) attribute twice; a
  // failure leaves the bit clear, and the launch below then fails loudly (the caller checks
  // cudaGetLastError after every op).
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_mask.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES, CK, BF, WIN, IOB, CH, HF>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES) == cudaSuccess)
      attr_mask.fetch_or(bit, std::memory_order_release);
  }
  const int g_sms = num_sms(dev);
  const int n_tiles = p.m_tiles * ((p.nout + BN - 1) / BN);
  const int grid = n_tiles < g_sms ? n_tiles : g_sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Roles<HF>::NT);
  cfg.dynamicSmemBytes = L::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, conv_tc_kernel<BN, STAGES, CK, BF, WIN, IOB, CH, HF>, ma, mw, mo, mr, p);
}

template <int IOB>
void launch_bf16(const CUtensorMap& map_a, const CUtensorMap& map_w, const CUtensorMap& map_out,
                 const CUtensorMap& map_res, const TcParams& p, cudaStream_t st) {
  if (p.win) {  // every tap from one bf16 window copy (SS MMAs at a row offset)
    switch (p.BN) {
      case 32: launch_bn<32, 12, 4, true, true, IOB>(map_a, map_w, map_out, map_res, p, st); break;
      case 64: launch_bn<64, 10, 4, true, true, IOB>(map_a, map_w, map_out, map_res, p, st); break;
      default:
        if (p.chain)
          launch_bn<128, 8, 4, true, true, IOB, true>(map_a, map_w, map_out, map_res, p, st);
        else
          launch_bn<128, 8, 4, true, true, IOB>(map_a, map_w, map_out, map_res, p, st);
        break;
    }
    return;
  }
  switch (p.BN) {
    case 32: launch_bn<32, 10, 4, true, false, IOB>(map_a, map_w, map_out, map_res, p, st); break;
    case 64: launch_bn<64, 8, 4, true, false, IOB>(map_a, map_w, map_out, map_res, p, st); break;
    default:
      if (p.chain)  // k3 conv + chained 1x1 conv in one launch
        launch_bn<128, 6, 4, true, false, IOB, true>(map_a, map_w, map_out, map_res, p, st);
      else
        launch_bn<128, 6, 4, true, false, IOB>(map_a, map_w, map_out, map_res, p, st);
      break;
  }
}

}  // namespace

void tc_trace_dump(long long* host) { cudaMemcpyFromSymbol(host, g_tc_trace, sizeof(long long) * 32 * 256); }

void launch_conv_tc(const CUtensorMap& map_a, const CUtensorMap& map_w, const CUtensorMap& map_out,
                    const CUtensorMap& map_res, const TcParams& p, cudaStream_t st) {
  // <BN, STAGES, CK (K-blocks per drained chunk), bf16, window, bf16 I/O>: as many stages as
  // shared memory holds next to the staging tile (narrow tiles are TMA-latency bound)
  if (p.bf16) {
    const int iob = (p.a_bf ? 1 : 0) | (p.o_bf ? 2 : 0);
    switch (iob) {
      case 0: launch_bf16<0>(map_a, map_w, map_out, map_res, p, st); break;
      case 1: launch_bf16<1>(map_a, map_w, map_out, map_res, p, st); break;
      case 2: launch_bf16<2>(map_a, map_w, map_out, map_res, p, st); break;
      default: launch_bf16<3>(map_a, map_w, map_out, map_res, p, st); break;
    }
    return;
  }
  if (p.f16) {  // 3xFP16 (HF): fp16 hi / lo planes, per-row power-of-two block scaling
    if (p.win) {
      switch (p.BN) {
        case 32: launch_bn<32, 14, 1, false, true, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
        case 64: launch_bn<64, 7, 1, false, true, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
        default: launch_bn<128, 4, 1, false, true, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
      }
      return;
    }
    switch (p.BN) {
      case 32: launch_bn<32, 16, 1, false, false, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
      case 64: launch_bn<64, 12, 1, false, false, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
      default: launch_bn<128, 4, 1, false, false, 0, false, true>(map_a, map_w, map_out, map_res, p, st); break;
    }
    return;
  }
  if (p.win) {  // narrow tiles, every tap from one window (see TcSmem); ring = weight region
    if (p.BN == 32)
      launch_bn<32, 14, 1, false, true>(map_a, map_w, map_out, map_res, p, st);
    else
      launch_bn<64, 7, 1, false, true>(map_a, map_w, map_out, map_res, p, st);
    return;
  }
  if (p.chain) {  // k3 conv + chained 1x1 conv in one launch (fp32, BN = 128)
    launch_bn<128, 3, 1, false, false, 0, true>(map_a, map_w, map_out, map_res, p, st);
    return;
  }
  switch (p.BN) {
    case 32: launch_bn<32, 8, 1, false>(map_a, map_w, map_out, map_res, p, st); break;
    case 64: launch_bn<64, 5, 1, false>(map_a, map_w, map_out, map_res, p, st); break;
    default: launch_bn<128, 3, 1, false>(map_a, map_w, map_out, map_res, p, st); break;
  }
}

}  // namespace scb
