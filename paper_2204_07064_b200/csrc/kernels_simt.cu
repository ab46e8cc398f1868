// kernels_simt.cu — bandwidth-class kernels of the streamconv B200 engine (sm_100a):
//   * conv_simt: generic cached frame-convolution on FFMA (narrow layers: PQMF, 16-channel
//     in/out convs, the gated head; and the fallback for shapes the tensor-core path does
//     not take).  Replaces conv1d (kernels.cpp:73-104) applied to concat(cache, buffer).
//   * ingest / egress: reference layout [stream][C][T] <-> frame-major buffers.
//   * carry: cached-padding update "keep the trailing N frames"
//     for every buffer and stream in ONE launch.
//   * reset_streams: SPEC reset for a subset of streams.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "kernels.hpp"

namespace scb {

namespace {

__device__ __forceinline__ float act_apply(float v, int kind, float alpha) {
  if (kind == ACT_LRELU) return v < 0.f ? alpha * v : v;  // kernels.cpp:125
  if (kind == ACT_TANH) return tanhf(v);                  // kernels.cpp:123
  return v;
}

// ------------------------------------------------------------------------ generic conv
// C tile BM x BN per CTA, BK=16 K-slab, 256 threads, TM x TN register micro-tile.
// K order is (tap, channel) ascending — fixed per layer, independent of T and of the number
// of streams, so outputs are bit-identical across buffer partitions.
template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) conv_simt_kernel(const ConvParams p) {
  constexpr int BK = 16;
  constexpr int NT = (BM / TM) * (BN / TN);
  static_assert(NT == 256, "256 threads");
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BN * BK / NT;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];

  const int tid = threadIdx.x;
  const int64_t M = static_cast<int64_t>(p.streams) * p.t_out;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int Ktot = p.taps * p.cin;

  // A loader: fixed column (k within slab) per thread, A_PER rows
  const int a_col = tid % BK;
  const int a_row0 = tid / BK;
  const float* a_ptr[A_PER];
#pragma unroll
  for (int e = 0; e < A_PER; ++e) {
    const int64_t m = m0 + a_row0 + e * (NT / BK);
    if (m < M) {
      const int64_t s = m / p.t_out;
      const int64_t i = m - s * p.t_out;
      a_ptr[e] = p.in + s * p.in_sstride +
                 (static_cast<int64_t>(p.in_f0) + i * p.row_step) * p.in_fstride + p.in_off;
    } else {
      a_ptr[e] = nullptr;
    }
  }
  const int64_t tap_stride = static_cast<int64_t>(p.tap_step) * p.in_fstride;

  const int tx = tid % (BN / TN);
  const int ty = tid / (BN / TN);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < Ktot; k0 += BK) {
    {
      const int kk = k0 + a_col;
      const int q = kk / p.cin;
      const int c = kk - q * p.cin;
      const bool kv = kk < Ktot;
#pragma unroll
      for (int e = 0; e < A_PER; ++e) {
        float v = 0.f;
        if (kv && a_ptr[e]) v = act_apply(__ldg(a_ptr[e] + q * tap_stride + c), p.pre_act, p.pre_alpha);
        As[a_col][a_row0 + e * (NT / BK)] = v;
      }
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = tid + e * NT;
      const int kr = idx / BN;
      const int nc = idx - kr * BN;
      const int kk = k0 + kr;
      const int n = n0 + nc;
      Bs[kr][nc] = (kk < Ktot && n < p.nout) ? __ldg(p.w + static_cast<int64_t>(kk) * p.nout + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[k][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  // epilogue: bias -> post-activation -> (gate) -> + residual -> store
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty * TM + i;
    if (m >= M) continue;
    const int64_t s = m / p.t_out;
    const int64_t row = m - s * p.t_out;
    float* orow = p.out + s * p.out_sstride + p.out_base + row * p.out_rstride;
    const float* rrow = p.res ? p.res + s * p.res_sstride +
                                    (static_cast<int64_t>(p.res_f0) + row) * p.res_fstride + p.res_off
                              : nullptr;
    if (p.gate) {
#pragma unroll
      for (int j = 0; j < TN; j += 2) {
        const int n = n0 + tx * TN + j;
        if (n >= p.nout) continue;
        const float a = acc[i][j] + __ldg(p.bias + n);
        const float g = acc[i][j + 1] + __ldg(p.bias + n + 1);
        orow[n >> 1] = tanhf(a) * (1.0f / (1.0f + expf(-g)));
      }
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = n0 + tx * TN + j;
        if (n >= p.nout) continue;
        float v = act_apply(acc[i][j] + __ldg(p.bias + n), p.post_act, p.post_alpha);
        if (rrow) v = v + act_apply(rrow[n], p.res_act, p.res_alpha);
        orow[n] = v;
      }
    }
  }
}

// ------------------------------------------------------------------------ ingest / egress
// Transposes run in 32-channel x 64-frame tiles: float4 loads/stores along the contiguous
// axis on both sides (frame rows of C floats in the buffer, time rows of T floats outside).
constexpr int TT = 64, TC = 32;

// Activation buffers are fp32 or (bf16 plans, tensor-core-only buffers) bf16.  `so` is the
// stream offset in 4-byte words (the buffer strides are kept in words either way); element
// (row, c) of a row of `fs` elements.
__device__ __forceinline__ void bput(float* buf, int bf, int64_t so, int64_t row, int fs, int c, float v) {
  if (bf)
    reinterpret_cast<__nv_bfloat16*>(buf)[2 * so + row * fs + c] = __float2bfloat16_rn(v);
  else
    buf[so + row * fs + c] = v;
}
__device__ __forceinline__ void bput4(float* buf, int bf, int64_t so, int64_t row, int fs, int c, float4 v) {
  if (bf) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(buf) + 2 * so + row * fs + c) = u;
  } else {
    *reinterpret_cast<float4*>(buf + so + row * fs + c) = v;
  }
}
__device__ __forceinline__ float bget(const float* buf, int bf, int64_t so, int64_t row, int fs, int c) {
  if (bf) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(buf)[2 * so + row * fs + c]);
  return buf[so + row * fs + c];
}
__device__ __forceinline__ float4 bget4(const float* buf, int bf, int64_t so, int64_t row, int fs, int c) {
  if (bf) {
    const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(buf) + 2 * so + row * fs + c);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  return *reinterpret_cast<const float4*>(buf + so + row * fs + c);
}

__global__ void __launch_bounds__(256) ingest_kernel(const IngestArgs a) {
  if (a.C == 1) {  // mono: contiguous copy per stream (float4 reads when aligned)
    if (a.T % 4 == 0 && (reinterpret_cast<uintptr_t>(a.in) & 15) == 0) {
      const int64_t total4 = static_cast<int64_t>(a.streams) * a.T / 4;
      for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total4;
           g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = (4 * g) / a.T, t = 4 * g - s * a.T;
        const float4 v = reinterpret_cast<const float4*>(a.in)[g];
        bput(a.buf, a.bf, s * a.sstride, a.cache + t, 1, 0, v.x);
        bput(a.buf, a.bf, s * a.sstride, a.cache + t + 1, 1, 0, v.y);
        bput(a.buf, a.bf, s * a.sstride, a.cache + t + 2, 1, 0, v.z);
        bput(a.buf, a.bf, s * a.sstride, a.cache + t + 3, 1, 0, v.w);
      }
      return;
    }
    const int64_t total = static_cast<int64_t>(a.streams) * a.T;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t s = g / a.T, t = g - s * a.T;
      bput(a.buf, a.bf, s * a.sstride, a.cache + t, 1, 0, a.in[g]);
    }
    return;
  }
  if (a.T < 16) {  // few frames per call (e.g. one latent frame): frame-major order, coalesced writes
    const int64_t total = static_cast<int64_t>(a.streams) * a.T * a.C;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t row = g / a.C;
      const int c = static_cast<int>(g - row * a.C);
      const int64_t s = row / a.T;
      const int t = static_cast<int>(row - s * a.T);
      bput(a.buf, a.bf, s * a.sstride, a.cache + t, a.C, c, a.in[(s * a.C + c) * a.T + t]);
    }
    return;
  }
  __shared__ float tile[TC][TT + 1];
  const bool in16 = (reinterpret_cast<uintptr_t>(a.in) & 15) == 0;  // caller's pointer
  if (a.C % 4 == 0 && a.C < TC && a.T % 4 == 0 && in16) {
    // narrow buffers (4..28 channels): tiles of all C channels x 2048/C frames, float4 on both
    // sides (a 32-channel tile would be mostly empty and fall back to scalar accesses)
    float* t2 = &tile[0][0];
    const int TTs = TC * TT / a.C, LD = TTs + 1, ntt = (a.T + TTs - 1) / TTs;
    const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt;
    const int tid = threadIdx.x, nv = a.C * TTs / 4, c4n = a.C / 4;
    for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
      const int64_t s = tile_id / ntt;
      const int t0 = static_cast<int>(tile_id - s * ntt) * TTs;
      const int tn = min(TTs, a.T - t0);
      for (int e = tid; e < nv; e += 256) {
        const int c = e / (TTs / 4), t4 = e - c * (TTs / 4);
        if (4 * t4 < tn) {
          const float4 v = *reinterpret_cast<const float4*>(a.in + (s * a.C + c) * a.T + t0 + 4 * t4);
          t2[c * LD + 4 * t4] = v.x;
          t2[c * LD + 4 * t4 + 1] = v.y;
          t2[c * LD + 4 * t4 + 2] = v.z;
          t2[c * LD + 4 * t4 + 3] = v.w;
        }
      }
      __syncthreads();
      for (int e = tid; e < tn * c4n; e += 256) {
        const int t = e / c4n, c4 = e - t * c4n;
        const float4 v = make_float4(t2[(4 * c4) * LD + t], t2[(4 * c4 + 1) * LD + t], t2[(4 * c4 + 2) * LD + t],
                                     t2[(4 * c4 + 3) * LD + t]);
        bput4(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.C, 4 * c4, v);
      }
      __syncthreads();
    }
    return;
  }
  const bool vec = (a.T % 4 == 0) && (a.C % 4 == 0) && in16;
  const int ntt = (a.T + TT - 1) / TT, ntc = (a.C + TC - 1) / TC;
  const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt * ntc;
  const int tid = threadIdx.x;
  for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
    const int64_t s = tile_id / (ntt * ntc);
    const int rem = static_cast<int>(tile_id - s * ntt * ntc);
    const int t0 = (rem / ntc) * TT, c0 = (rem % ntc) * TC;
    const bool full = vec && t0 + TT <= a.T && c0 + TC <= a.C;
    if (full) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = tid + 256 * k;      // 512 float4 = 32 channel rows x 16
        const int c = e >> 4, t4 = e & 15;
        const float4 v = *reinterpret_cast<const float4*>(a.in + (s * a.C + c0 + c) * a.T + t0 + 4 * t4);
        tile[c][4 * t4] = v.x;
        tile[c][4 * t4 + 1] = v.y;
        tile[c][4 * t4 + 2] = v.z;
        tile[c][4 * t4 + 3] = v.w;
      }
    } else {
      for (int e = tid; e < TC * TT; e += 256) {
        const int c = e / TT, t = e % TT;
        tile[c][t] = (c0 + c < a.C && t0 + t < a.T) ? a.in[(s * a.C + c0 + c) * a.T + t0 + t] : 0.f;
      }
    }
    __syncthreads();
    if (full) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = tid + 256 * k;      // 512 float4 = 64 frames x 8
        const int t = e >> 3, c4 = e & 7;
        const float4 v = make_float4(tile[4 * c4][t], tile[4 * c4 + 1][t], tile[4 * c4 + 2][t], tile[4 * c4 + 3][t]);
        bput4(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.C, c0 + 4 * c4, v);
      }
    } else {
      for (int e = tid; e < TC * TT; e += 256) {
        const int t = e / TC, c = e % TC;
        if (t0 + t < a.T && c0 + c < a.C)
          bput(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.C, c0 + c, tile[c][t]);
      }
    }
    __syncthreads();
  }
}

// Wide sources (C a multiple of TCH = 32 or 16, T a multiple of 4096 / TCH, aligned): tiles of
// TCH channels x 4096 / TCH frames, the channel rows read with all of a thread's four float4
// loads in flight before the barrier (ingest_kernel's 64-frame tiles keep two).
template <int TCH>
__global__ void __launch_bounds__(256) ingest_wide_kernel(const IngestArgs a) {
  constexpr int FR = 4096 / TCH, R4 = FR / 4, C4 = TCH / 4;
  __shared__ float it_[TCH][FR + 1];
  const int ntt = a.T / FR, ntc = a.C / TCH;
  const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt * ntc;
  const int tid = threadIdx.x;
  for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
    const int64_t s = tile_id / (ntt * ntc);
    const int rem = static_cast<int>(tile_id - s * ntt * ntc);
    const int t0 = (rem / ntc) * FR, c0 = (rem % ntc) * TCH;
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 1024 float4 = TCH channel rows x FR / 4
      const int e = tid + 256 * k;
      v[k] = *reinterpret_cast<const float4*>(a.in + (s * a.C + c0 + e / R4) * a.T + t0 + 4 * (e % R4));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = tid + 256 * k;
      const int c = e / R4, t4 = e % R4;
      it_[c][4 * t4] = v[k].x;
      it_[c][4 * t4 + 1] = v[k].y;
      it_[c][4 * t4 + 2] = v[k].z;
      it_[c][4 * t4 + 3] = v[k].w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 1024 float4 = FR frames x TCH / 4
      const int e = tid + 256 * k;
      const int t = e / C4, c4 = e % C4;
      bput4(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.C, c0 + 4 * c4,
            make_float4(it_[4 * c4][t], it_[4 * c4 + 1][t], it_[4 * c4 + 2][t], it_[4 * c4 + 3][t]));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) egress_kernel(const EgressArgs a) {
  if (a.C == 1) {
    if (a.T % 4 == 0 && a.fstride == 1 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0) {  // float4 writes
      const int64_t total4 = static_cast<int64_t>(a.streams) * a.T / 4;
      for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total4;
           g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = (4 * g) / a.T, t = 4 * g - s * a.T;
        const int64_t so = s * a.sstride;
        reinterpret_cast<float4*>(a.out)[g] =
            make_float4(act_apply(bget(a.buf, a.bf, so, a.cache + t, 1, a.off), a.act, a.alpha),
                        act_apply(bget(a.buf, a.bf, so, a.cache + t + 1, 1, a.off), a.act, a.alpha),
                        act_apply(bget(a.buf, a.bf, so, a.cache + t + 2, 1, a.off), a.act, a.alpha),
                        act_apply(bget(a.buf, a.bf, so, a.cache + t + 3, 1, a.off), a.act, a.alpha));
      }
      return;
    }
    const int64_t total = static_cast<int64_t>(a.streams) * a.T;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t s = g / a.T, t = g - s * a.T;
      a.out[g] = act_apply(bget(a.buf, a.bf, s * a.sstride, a.cache + t, a.fstride, a.off), a.act, a.alpha);
    }
    return;
  }
  __shared__ float tile[TC][TT + 1];
  const bool out16 = (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;  // caller's pointer
  if (a.C % 4 == 0 && a.C < TC && a.T % 4 == 0 && a.fstride % 4 == 0 && a.off % 4 == 0 && out16) {
    // narrow sinks: all C channels x 2048/C frames per tile (see ingest_kernel)
    float* t2 = &tile[0][0];
    const int TTs = TC * TT / a.C, LD = TTs + 1, ntt = (a.T + TTs - 1) / TTs;
    const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt;
    const int tid = threadIdx.x, nv = a.C * TTs / 4, c4n = a.C / 4;
    for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
      const int64_t s = tile_id / ntt;
      const int t0 = static_cast<int>(tile_id - s * ntt) * TTs;
      const int tn = min(TTs, a.T - t0);
      for (int e = tid; e < tn * c4n; e += 256) {
        const int t = e / c4n, c4 = e - t * c4n;
        const float4 v = bget4(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.fstride, a.off + 4 * c4);
        t2[(4 * c4) * LD + t] = act_apply(v.x, a.act, a.alpha);
        t2[(4 * c4 + 1) * LD + t] = act_apply(v.y, a.act, a.alpha);
        t2[(4 * c4 + 2) * LD + t] = act_apply(v.z, a.act, a.alpha);
        t2[(4 * c4 + 3) * LD + t] = act_apply(v.w, a.act, a.alpha);
      }
      __syncthreads();
      for (int e = tid; e < nv; e += 256) {
        const int c = e / (TTs / 4), t4 = e - c * (TTs / 4);
        if (4 * t4 < tn)
          *reinterpret_cast<float4*>(a.out + (s * a.C + c) * a.T + t0 + 4 * t4) =
              make_float4(t2[c * LD + 4 * t4], t2[c * LD + 4 * t4 + 1], t2[c * LD + 4 * t4 + 2], t2[c * LD + 4 * t4 + 3]);
      }
      __syncthreads();
    }
    return;
  }
  const bool vec = (a.T % 4 == 0) && (a.C % 4 == 0) && (a.fstride % 4 == 0) && (a.off % 4 == 0) && out16;
  const int ntt = (a.T + TT - 1) / TT, ntc = (a.C + TC - 1) / TC;
  const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt * ntc;
  const int tid = threadIdx.x;
  for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
    const int64_t s = tile_id / (ntt * ntc);
    const int rem = static_cast<int>(tile_id - s * ntt * ntc);
    const int t0 = (rem / ntc) * TT, c0 = (rem % ntc) * TC;
    const bool full = vec && t0 + TT <= a.T && c0 + TC <= a.C;
    if (full) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = tid + 256 * k;
        const int t = e >> 3, c4 = e & 7;
        const float4 v = bget4(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.fstride, a.off + c0 + 4 * c4);
        tile[4 * c4][t] = act_apply(v.x, a.act, a.alpha);
        tile[4 * c4 + 1][t] = act_apply(v.y, a.act, a.alpha);
        tile[4 * c4 + 2][t] = act_apply(v.z, a.act, a.alpha);
        tile[4 * c4 + 3][t] = act_apply(v.w, a.act, a.alpha);
      }
    } else {
      for (int e = tid; e < TC * TT; e += 256) {
        const int t = e / TC, c = e % TC;
        tile[c][t] = (t0 + t < a.T && c0 + c < a.C)
                         ? act_apply(bget(a.buf, a.bf, s * a.sstride, a.cache + t0 + t, a.fstride, a.off + c0 + c),
                                     a.act, a.alpha)
                         : 0.f;
      }
    }
    __syncthreads();
    if (full) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = tid + 256 * k;
        const int c = e >> 4, t4 = e & 15;
        const float4 v = make_float4(tile[c][4 * t4], tile[c][4 * t4 + 1], tile[c][4 * t4 + 2], tile[c][4 * t4 + 3]);
        *reinterpret_cast<float4*>(a.out + (s * a.C + c0 + c) * a.T + t0 + 4 * t4) = v;
      }
    } else {
      for (int e = tid; e < TC * TT; e += 256) {
        const int c = e / TT, t = e % TT;
        if (c0 + c < a.C && t0 + t < a.T) a.out[(s * a.C + c0 + c) * a.T + t0 + t] = tile[c][t];
      }
    }
    __syncthreads();
  }
}

// Wide sinks (C a multiple of TCH = 32 or 16, T a multiple of 4096 / TCH, aligned): tiles of
// TCH channels x 4096 / TCH frames, 4 float4 per thread each side with the loads issued first
// — more bytes in flight per barrier than egress_kernel's 64-frame tiles, and long channel-
// major rows on the write side.  Kernels of their own so the general paths keep their
// register budget.
template <int TCH>
__global__ void __launch_bounds__(256) egress_wide_kernel(const EgressArgs a) {
  constexpr int FR = 4096 / TCH, R4 = FR / 4, C4 = TCH / 4;
  __shared__ float et[TCH][FR + 1];
  const int ntt = a.T / FR, ntc = a.C / TCH;
  const int64_t ntiles = static_cast<int64_t>(a.streams) * ntt * ntc;
  const int tid = threadIdx.x;
  for (int64_t tile_id = blockIdx.x; tile_id < ntiles; tile_id += gridDim.x) {
    const int64_t s = tile_id / (ntt * ntc);
    const int rem = static_cast<int>(tile_id - s * ntt * ntc);
    const int t0 = (rem / ntc) * FR, c0 = (rem % ntc) * TCH;
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = tid + 256 * k;
      v[k] = bget4(a.buf, a.bf, s * a.sstride, a.cache + t0 + e / C4, a.fstride, a.off + c0 + 4 * (e % C4));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = tid + 256 * k;
      const int t = e / C4, c4 = e % C4;
      et[4 * c4][t] = act_apply(v[k].x, a.act, a.alpha);
      et[4 * c4 + 1][t] = act_apply(v[k].y, a.act, a.alpha);
      et[4 * c4 + 2][t] = act_apply(v[k].z, a.act, a.alpha);
      et[4 * c4 + 3][t] = act_apply(v[k].w, a.act, a.alpha);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = tid + 256 * k;
      const int c = e / R4, t4 = e % R4;
      *reinterpret_cast<float4*>(a.out + (s * a.C + c0 + c) * a.T + t0 + 4 * t4) =
          make_float4(et[c][4 * t4], et[c][4 * t4 + 1], et[c][4 * t4 + 2], et[c][4 * t4 + 3]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------ carry / reset
// One thread per (buffer, stream, channel column).  Frames move in ascending order in chunks
// of 8 (all loads of a chunk before its stores): a chunk never reads a frame a previous
// store wrote, because every load index f+T+u exceeds every earlier store index (T >= 1).
__global__ void carry_kernel(const BufDesc* __restrict__ bufs, int nbuf, int streams, int64_t items) {
  __shared__ BufDesc sb[64];
  for (int i = threadIdx.x; i < nbuf; i += blockDim.x) sb[i] = bufs[i];
  __syncthreads();
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < items;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int b = 0;
    while (b + 1 < nbuf && sb[b + 1].item0 <= g) ++b;
    const BufDesc d = sb[b];
    const int64_t loc = g - d.item0;
    const int64_t T = d.t;
    if ((d.C & 3) == 0) {  // float4 column groups: 16 B per thread, 512 B per warp and row
      const int G = d.C >> 2;
      const int64_t s = loc / G;
      const int c4 = static_cast<int>(loc - s * G);
      float4* col = reinterpret_cast<float4*>(d.base + s * d.sstride) + c4;
      const int64_t fs = G;
      int f = 0;
      for (; f + 8 <= d.cache; f += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = col[(f + u + T) * fs];
#pragma unroll
        for (int u = 0; u < 8; ++u) col[(f + u) * fs] = v[u];
      }
      for (; f < d.cache; ++f) col[f * fs] = col[(f + T) * fs];
      continue;
    }
    const int64_t s = loc / d.C;
    const int c = static_cast<int>(loc - s * d.C);
    float* col = d.base + s * d.sstride + c;
    const int64_t fs = d.C;
    int f = 0;
    for (; f + 8 <= d.cache; f += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = col[(f + u + T) * fs];
#pragma unroll
      for (int u = 0; u < 8; ++u) col[(f + u) * fs] = v[u];
    }
    for (; f < d.cache; ++f) col[f * fs] = col[(f + T) * fs];
  }
  (void)streams;
}

__global__ void reset_streams_kernel(const BufDesc* __restrict__ bufs, int nbuf,
                                     const int* __restrict__ ids, int n_ids, int64_t per_stream) {
  __shared__ BufDesc sb[64];
  for (int i = threadIdx.x; i < nbuf; i += blockDim.x) sb[i] = bufs[i];
  __syncthreads();
  const int64_t items = per_stream * n_ids;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < items;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = g / per_stream;
    const int64_t r = g - k * per_stream;
    int b = 0;
    while (b + 1 < nbuf && sb[b + 1].ritem0 <= r) ++b;
    const BufDesc d = sb[b];
    const int c = static_cast<int>(r - d.ritem0);
    float* col = d.base + static_cast<int64_t>(ids[k]) * d.sstride + c;
    for (int f = 0; f < d.cache; ++f) col[static_cast<int64_t>(f) * d.C] = 0.f;
  }
}

// reference Kernel weights [N][M][K] -> [K][M][N] (the generic conv's B layout)
__global__ void relayout_w_kernel(const float* __restrict__ w, int N, int M, int K,
                                  float* __restrict__ o) {
  const int64_t total = static_cast<int64_t>(N) * M * K;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = g / (static_cast<int64_t>(M) * K);
    const int64_t r = g - n * M * K;
    const int64_t m = r / K, k = r - m * K;
    o[(k * M + m) * N + n] = w[g];
  }
}

// SPEC Sum over frame-major buffers (kernels.hpp SumParams): one thread per output element,
// consecutive threads on consecutive channels of a frame (coalesced rows in and out).
__global__ void __launch_bounds__(256) sum_kernel(const SumParams p) {
  const int64_t total = static_cast<int64_t>(p.streams) * p.t_out * p.C;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % p.C);
    const int64_t st = e / p.C;
    const int t = static_cast<int>(st % p.t_out);
    const int64_t s = st / p.t_out;
    float acc = 0.f;
#pragma unroll
    for (int q = 0; q < kMaxSumIn; ++q) {
      if (q >= p.n_in) break;
      const float v = act_apply(
          p.in[q][s * p.in_sstride[q] + static_cast<int64_t>(p.in_f0[q] + t) * p.in_fstride[q] + p.in_off[q] + c],
          p.act[q], p.alpha[q]);
      acc = (q == 0) ? v : acc + v;  // left to right in port order, like the oracle's Sum
    }
    p.out[s * p.out_sstride + p.out_base + static_cast<int64_t>(t) * p.C + c] =
        act_apply(acc, p.post_act, p.post_alpha);
  }
}

__global__ void __launch_bounds__(256) cast_kernel(uint16_t* bf, float* f, int64_t n, int to_f32) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (to_f32)
      f[i] = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bf)[i]);
    else
      reinterpret_cast<__nv_bfloat16*>(bf)[i] = __float2bfloat16_rn(f[i]);
  }
}

int grid_for(int64_t items, int threads) {
  int64_t g = (items + threads - 1) / threads;
  const int64_t cap = 148 * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

const void* ingest_kernel_ptr() { return reinterpret_cast<const void*>(&ingest_kernel); }
const void* egress_kernel_ptr() { return reinterpret_cast<const void*>(&egress_kernel); }
bool is_egress_wide_kernel(const void* f) {
  return f == reinterpret_cast<const void*>(&egress_wide_kernel<32>) ||
         f == reinterpret_cast<const void*>(&egress_wide_kernel<16>);
}
bool is_ingest_wide_kernel(const void* f) {
  return f == reinterpret_cast<const void*>(&ingest_wide_kernel<32>) ||
         f == reinterpret_cast<const void*>(&ingest_wide_kernel<16>);
}

// channels per wide tile (0: the general kernel)
int wide_tch(int C, int T) {
  if (C % 32 == 0 && T % 128 == 0) return 32;
  if (C % 16 == 0 && T % 256 == 0) return 16;
  return 0;
}

bool ingest_wide(const IngestArgs& a) {
  return wide_tch(a.C, a.T) > 0 && (reinterpret_cast<uintptr_t>(a.in) & 15) == 0;
}

bool egress_wide(const EgressArgs& a) {
  return wide_tch(a.C, a.T) > 0 && a.fstride % 4 == 0 && a.off % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
}

void launch_ingest(const IngestArgs& a, cudaStream_t st) {
  if (ingest_wide(a)) {
    const int tch = wide_tch(a.C, a.T);
    const int64_t tiles = static_cast<int64_t>(a.streams) * (a.T / (4096 / tch)) * (a.C / tch);
    if (tch == 32)
      ingest_wide_kernel<32><<<grid_for(tiles, 1), 256, 0, st>>>(a);
    else
      ingest_wide_kernel<16><<<grid_for(tiles, 1), 256, 0, st>>>(a);
    return;
  }
  if (a.C == 1) {
    ingest_kernel<<<grid_for(static_cast<int64_t>(a.streams) * a.T, 256), 256, 0, st>>>(a);
  } else if (a.T < 16) {
    ingest_kernel<<<grid_for(static_cast<int64_t>(a.streams) * a.T * a.C, 256), 256, 0, st>>>(a);
  } else {
    // grid for the generic tiling (the kernel loops over its tiles persistently either way)
    const int64_t tiles = static_cast<int64_t>(a.streams) * ((a.T + TT - 1) / TT) * ((a.C + TC - 1) / TC);
    ingest_kernel<<<grid_for(tiles, 1), 256, 0, st>>>(a);
  }
}

void launch_egress(const EgressArgs& a, cudaStream_t st) {
  if (egress_wide(a)) {
    const int tch = wide_tch(a.C, a.T);
    const int64_t tiles = static_cast<int64_t>(a.streams) * (a.T / (4096 / tch)) * (a.C / tch);
    if (tch == 32)
      egress_wide_kernel<32><<<grid_for(tiles, 1), 256, 0, st>>>(a);
    else
      egress_wide_kernel<16><<<grid_for(tiles, 1), 256, 0, st>>>(a);
    return;
  }
  if (a.C == 1) {
    egress_kernel<<<grid_for(static_cast<int64_t>(a.streams) * a.T, 256), 256, 0, st>>>(a);
  } else {
    const int64_t tiles = static_cast<int64_t>(a.streams) * ((a.T + TT - 1) / TT) * ((a.C + TC - 1) / TC);
    egress_kernel<<<grid_for(tiles, 1), 256, 0, st>>>(a);
  }
}

void launch_conv_simt(const ConvParams& p, cudaStream_t st) {
  const int64_t M = static_cast<int64_t>(p.streams) * p.t_out;
  if (p.nout > 32) {
    dim3 grid(static_cast<unsigned>((M + 63) / 64), (p.nout + 63) / 64);
    conv_simt_kernel<64, 64, 4, 4><<<grid, 256, 0, st>>>(p);
  } else if (p.nout > 16) {
    dim3 grid(static_cast<unsigned>((M + 127) / 128), (p.nout + 31) / 32);
    conv_simt_kernel<128, 32, 4, 4><<<grid, 256, 0, st>>>(p);
  } else {
    dim3 grid(static_cast<unsigned>((M + 255) / 256), (p.nout + 15) / 16);
    conv_simt_kernel<256, 16, 4, 4><<<grid, 256, 0, st>>>(p);
  }
}

void launch_cast(uint16_t* bf, float* f, int64_t n, bool to_f32, cudaStream_t st) {
  if (n <= 0) return;
  cast_kernel<<<grid_for(n, 256), 256, 0, st>>>(bf, f, n, to_f32 ? 1 : 0);
}

void launch_sum(const SumParams& p, cudaStream_t st) {
  if (p.t_out <= 0 || p.streams <= 0) return;
  sum_kernel<<<grid_for(static_cast<int64_t>(p.streams) * p.t_out * p.C, 256), 256, 0, st>>>(p);
}

void launch_carry(const BufDesc* d_bufs, int nbuf, int streams, int64_t items, cudaStream_t st) {
  if (nbuf == 0 || items == 0) return;
  carry_kernel<<<grid_for(items, 256), 256, 0, st>>>(d_bufs, nbuf, streams, items);
}

void launch_relayout_w(const float* w, int N, int M, int K, float* o, cudaStream_t st) {
  relayout_w_kernel<<<grid_for(static_cast<int64_t>(N) * M * K, 256), 256, 0, st>>>(w, N, M, K, o);
}

void launch_reset_streams(const BufDesc* d_bufs, int nbuf, const int* d_ids, int n_ids,
                          int64_t per_stream, cudaStream_t st) {
  if (nbuf == 0 || n_ids == 0 || per_stream == 0) return;
  reset_streams_kernel<<<grid_for(per_stream * n_ids, 256), 256, 0, st>>>(d_bufs, nbuf, d_ids,
                                                                           n_ids, per_stream);
}

}  // namespace scb
