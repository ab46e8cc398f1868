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
// activation split (and the fused pre-activation LeakyReLU/tanh) is done in shared memory by
// the transform warps between the TMA landing and the MMA issue — elementwise, so it is
// oblivious to the 128B swizzle.
//
// The tensor core accumulates in fp32 with truncation, so long K loops drift (measured: ~4e-5
// x RMS per layer at K=384..1536).  The MMA therefore accumulates only CK K-blocks (a chunk)
// into one of two TMEM buffers — the main A_hi W_hi product and the two small correction
// products in separate accumulators — and the drain warps add each chunk into fp32
// registers with round-to-nearest adds (fixed order, independent of T and of the stream
// count), which keeps the path at FFMA-level accuracy at any depth.
//
// Persistent: grid = #SMs, static tile striding; the TMA/transform/MMA pipeline runs across
// tile boundaries and the drain/epilogue of tile t overlaps the MMAs of tile t+1.
// Warp roles (480 threads): w0 TMA producer | w1 TMEM alloc + single-thread MMA issuer |
// w2..w5 transform | w6..w13 drain + epilogue (TMEM lane quarter = warp % 4, column half =
// (warp - 6) / 4) | w14 epilogue I/O: residual tile TMA-loaded into the staging buffer as soon
// as the previous output store has read it, output tile TMA-stored from staging.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_tc.hpp"

namespace scb {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 per 128-byte swizzled row
constexpr uint32_t A_TILE = BM * BK * 4;  // 16 KB
constexpr int NUM_THREADS = 480;
constexpr int XF_WARP0 = 2;   // transform warps 2..5
constexpr int EP_WARP0 = 6;   // drain/epilogue warps 6..13
constexpr int IO_WARP = 14;   // residual TMA loads + output TMA stores

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

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
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
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float act_apply(float v, int kind, float alpha) {
  if (kind == ACT_LRELU) return v < 0.f ? alpha * v : v;
  if (kind == ACT_TANH) return tanhf(v);
  return v;
}

template <int BN, int STAGES>
struct TcSmem {
  static constexpr uint32_t B_TILE = BN * BK * 4;
  static constexpr uint32_t STAGE = 2 * A_TILE + 2 * B_TILE;
  static constexpr uint32_t STAGING = BM * BN * 4;  // residual-in / output-out tile, 32-col SW128 slabs
  static constexpr uint32_t BYTES = STAGES * STAGE + STAGING + 1024 /*barriers*/ + 8192 /*bias*/ + 1024;
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

template <int BN, int STAGES, int CK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
                   const __grid_constant__ CUtensorMap tmap_out, const __grid_constant__ CUtensorMap tmap_res,
                   const TcParams p) {
  using L = TcSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg = reinterpret_cast<float*>(smem + STAGES * L::STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE + L::STAGING);
  uint64_t* full = bars;
  uint64_t* xform = bars + STAGES;
  uint64_t* empty = bars + 2 * STAGES;
  uint64_t* tfull = bars + 3 * STAGES;       // [2]
  uint64_t* tempty = bars + 3 * STAGES + 2;  // [2]
  uint64_t* res_full = bars + 3 * STAGES + 4;
  uint64_t* stg_written = bars + 3 * STAGES + 5;
  uint64_t* stg_free = bars + 3 * STAGES + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 7);
  float* sbias = reinterpret_cast<float*>(smem + STAGES * L::STAGE + L::STAGING + 1024);  // <= 2048 floats

  auto a_hi = [&](int s) { return smem + s * L::STAGE; };
  auto a_lo = [&](int s) { return smem + s * L::STAGE + A_TILE; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE + 2 * A_TILE; };
  auto b_lo = [&](int s) { return smem + s * L::STAGE + 2 * A_TILE + L::B_TILE; };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = p.n_kblocks;
  const int n_tiles_n = (p.nout + BN - 1) / BN;
  const int n_tiles = p.m_tiles * n_tiles_n;
  constexpr uint32_t TMEM_COLS = (4 * BN < 32) ? 32 : 4 * BN;  // 2 buffers x (main, corr)

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xform[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    mbar_init(res_full, 1);
    mbar_init(stg_written, 8);
    mbar_init(stg_free, 1);
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
  for (int i = threadIdx.x; i < p.nout; i += NUM_THREADS) sbias[i] = p.bias[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(BK * 4 * p.R * p.G) + 2 * L::B_TILE;
      int g = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) + 1) & 1);
          const int q = kb / p.cblocks;
          const int cb = kb - q * p.cblocks;
          mbar_expect_tx(&full[s], bytes);
          tma_load_3d(&tmap_a, &full[s], a_hi(s), p.a_c0 + cb * BK, p.a_row0 + tc.i0 + q * p.a_tap_rows, tc.s0);
          tma_load_3d(&tmap_w, &full[s], b_hi(s), kb * BK, tc.n0, 0);
          tma_load_3d(&tmap_w, &full[s], b_lo(s), kb * BK, tc.n0, 1);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(BM >> 4) << 24);
      int g = 0, c = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          const int b = c & 1;
          const bool chunk_first = (kb % CK) == 0;
          const bool chunk_last = ((kb % CK) == CK - 1) || (kb == nk - 1);
          if (chunk_first && c >= 2) mbar_wait(&tempty[b], ((c >> 1) + 1) & 1);
          mbar_wait(&xform[s], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t dmain = tmem_base + static_cast<uint32_t>(b * 2 * BN);
          const uint32_t dcorr = dmain + BN;
          const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(s));
          const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
            const uint32_t acc0 = (!chunk_first || kk > 0) ? 1u : 0u;
            if (!(p.debug & 2)) {
              mma_tf32(dcorr, sw128_desc(al + off), sw128_desc(bh + off), idesc, acc0);
              mma_tf32(dcorr, sw128_desc(ah + off), sw128_desc(bl + off), idesc, 1u);
            }
            mma_tf32(dmain, sw128_desc(ah + off), sw128_desc(bh + off), idesc, acc0);
          }
          mma_commit(&empty[s]);
          if (chunk_last) {
            mma_commit(&tfull[b]);
            ++c;
          }
        }
      }
    }
  } else if (warp == IO_WARP) {
    // ===================== epilogue I/O (one thread) =====================
    if (lane == 0) {
      const int n_tiles_n2 = n_tiles_n;
      const int out_cols = p.gate ? BN / 2 : BN;
      int tcount = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        const TileCoord tc = tile_coord(p, tile, n_tiles_n2, BN);
        if (p.res) {  // staging is free (previous store read it): bring this tile's residual in
          mbar_expect_tx(res_full, static_cast<uint32_t>(BN / 32) * 32u * 4u * p.R * p.G);
          for (int k = 0; k < BN / 32; ++k)
            tma_load_3d(&tmap_res, res_full, stg + k * (BM * 32), p.res_off + tc.n0 + 32 * k, tc.i0, tc.s0);
        }
        if (p.debug & 8) continue;
        mbar_wait(stg_written, tcount & 1);
        const int oc0 = p.gate ? tc.n0 / 2 : tc.n0;
        for (int k = 0; k < (out_cols + 31) / 32; ++k)
          tma_store_3d(&tmap_out, stg + k * (BM * 32), oc0 + 32 * k, tc.i0, tc.s0);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(stg_free);
      }
      bulk_wait0();
    }
  } else if (warp < EP_WARP0) {
    // ===================== transform (w2..w5) =====================
    const int t = threadIdx.x - XF_WARP0 * 32;  // 0..127
    int g = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        float4* ah = reinterpret_cast<float4*>(a_hi(s));
        float4* al = reinterpret_cast<float4*>(a_lo(s));
#pragma unroll
        for (int j = 0; j < ((p.debug & 1) ? 0 : (BM * BK / 4) / 128); ++j) {
          const int e = t + j * 128;
          const float4 v = ah[e];
          float x[4] = {v.x, v.y, v.z, v.w};
          float h[4], l[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float a = act_apply(x[u], p.pre_act, p.pre_alpha);
            h[u] = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
            l[u] = a - h[u];
          }
          ah[e] = make_float4(h[0], h[1], h[2], h[3]);
          al[e] = make_float4(l[0], l[1], l[2], l[3]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xform[s]);
      }
    }
  } else {
    // ===================== drain + epilogue (w6..w13) =====================
    constexpr int COLS = BN / 2;
    const int quarter = warp & 3;
    const int half = (warp - EP_WARP0) >> 2;
    const int r = quarter * 32 + lane;  // tile row == TMEM lane
    const int col0 = half * COLS;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + col0;
    float acc[COLS];
#pragma unroll
    for (int u = 0; u < COLS; ++u) acc[u] = 0.f;
    int c = 0, tcount = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
      const TileCoord tc = tile_coord(p, tile, n_tiles_n, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const bool chunk_last = ((kb % CK) == CK - 1) || (kb == nk - 1);
        if (!chunk_last) continue;
        const bool first = (kb / CK) == 0;
        const int b = c & 1;
        mbar_wait(&tfull[b], (c >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < COLS; cc += 16) {
          uint32_t vm[16], vc[16];
          if (p.debug & 4) {
#pragma unroll
            for (int u = 0; u < 16; ++u) vm[u] = vc[u] = 0u;
          } else {
            tmem_ld16(lane_base + static_cast<uint32_t>(b * 2 * BN + cc), vm);
            tmem_ld16(lane_base + static_cast<uint32_t>(b * 2 * BN + BN + cc), vc);
            tmem_wait_ld();
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float x = __uint_as_float(vm[u]) + __uint_as_float(vc[u]);
            acc[cc + u] = first ? x : acc[cc + u] + x;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        ++c;
      }
      // ---- epilogue: bias/act/gate (+ residual from staging) -> staging (TMA-stored by w14)
      if (p.debug & 8) continue;
      if (p.res) {
        mbar_wait(res_full, tcount & 1);
      } else if (tcount > 0) {
        mbar_wait(stg_free, (tcount - 1) & 1);
      }
      if (p.gate) {
#pragma unroll
        for (int u = 0; u < COLS; u += 2) {
          const int n = tc.n0 + col0 + u;
          const float a = acc[u] + sbias[n];
          const float gg = acc[u + 1] + sbias[n + 1];
          stg[stg_off(r, (col0 + u) >> 1)] = tanhf(a) * (1.0f / (1.0f + expf(-gg)));
        }
      } else {
#pragma unroll
        for (int u = 0; u < COLS; u += 4) {
          const int n = tc.n0 + col0 + u;
          const float4 bv = *reinterpret_cast<const float4*>(sbias + n);
          float4* dst = reinterpret_cast<float4*>(stg + stg_off(r, col0 + u));
          float4 o;
          o.x = act_apply(acc[u] + bv.x, p.post_act, p.post_alpha);
          o.y = act_apply(acc[u + 1] + bv.y, p.post_act, p.post_alpha);
          o.z = act_apply(acc[u + 2] + bv.z, p.post_act, p.post_alpha);
          o.w = act_apply(acc[u + 3] + bv.w, p.post_act, p.post_alpha);
          if (p.res) {
            const float4 rv = *dst;
            o.x += act_apply(rv.x, p.res_act, p.res_alpha);
            o.y += act_apply(rv.y, p.res_act, p.res_alpha);
            o.z += act_apply(rv.z, p.res_act, p.res_alpha);
            o.w += act_apply(rv.w, p.res_act, p.res_alpha);
          }
          *dst = o;
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(stg_written);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

int g_num_sms = 0;

template <int BN, int STAGES, int CK>
void launch_bn(const CUtensorMap& ma, const CUtensorMap& mw, const CUtensorMap& mo, const CUtensorMap& mr,
               const TcParams& p, cudaStream_t st) {
  using L = TcSmem<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    attr = true;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int n_tiles = p.m_tiles * ((p.nout + BN - 1) / BN);
  const int grid = n_tiles < g_num_sms ? n_tiles : g_num_sms;
  conv_tc_kernel<BN, STAGES, CK><<<grid, NUM_THREADS, L::BYTES, st>>>(ma, mw, mo, mr, p);
}

}  // namespace

void launch_conv_tc(const CUtensorMap& map_a, const CUtensorMap& map_w, const CUtensorMap& map_out,
                    const CUtensorMap& map_res, const TcParams& p, cudaStream_t st) {
  switch (p.BN) {
    case 32: launch_bn<32, 4, 1>(map_a, map_w, map_out, map_res, p, st); break;
    case 64: launch_bn<64, 3, 1>(map_a, map_w, map_out, map_res, p, st); break;
    default: launch_bn<128, 2, 1>(map_a, map_w, map_out, map_res, p, st); break;
  }
}

}  // namespace scb
