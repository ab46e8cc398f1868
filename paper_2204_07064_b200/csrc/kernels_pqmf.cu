// kernels_pqmf.cu — PQMF analysis / synthesis in the polyphase + cosine-modulation form.
//
// A 16-band, 256-tap pseudo-QMF bank as plain convolutions costs 256 MACs per sample (the
// generic conv path).  Its weights are a prototype modulated by cosines that repeat every 2M
// taps, so (factorisation verified at plan time, graph.cpp factor_pqmf_*):
//   analysis : y[n] = bias[n] + sum_b Cm[n][b] * u[b],  u[b] = sum_a S[a][b] * x[2M a + b]
//              (8 x 32 + 16 x 32 = 768 MACs per 16-sample frame = 48 per sample)
//   synthesis: V[t][k] = sum_c R[k][c] x[t][c] (one modulation per input frame, NCLS classes),
//              y[M i + ph] = bias + sum_q s[q][ph] * V[i + q][class(q, ph)]
//              with class(q, ph) = (q mod P) * Mh + (mirror ? min(ph, M-1-ph) : ph) after the
//              plan-time canonical renumbering (16 classes for the symmetric prototype: 16 + 16
//              MACs per sample).
// Both read the input once from HBM (staged in shared memory) and write the output once; the
// inner loops are shared-memory-read bound, so the layouts below keep every warp access
// conflict-free and vectorise the broadcast coefficient reads.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_pqmf.hpp"

namespace scb {

namespace {

constexpr int M = 16;      // bands
constexpr int B = 32;      // 2M modulation phases
static_assert(sizeof(PqmfCoef) + sizeof(PqmfParams) <= 4000, "coefficients fit the 4 KB parameter bank");
constexpr int A = 8;       // prototype phases (taps / 2M)
constexpr int K = A * B;   // 256 taps
constexpr int Q = 16;      // synthesis taps over input frames (K / M)
constexpr int FB = 128;    // output rows per block (= threads)

__device__ __forceinline__ float act_apply(float v, int kind, float alpha) {
  if (kind == ACT_LRELU) return v < 0.f ? alpha * v : v;
  if (kind == ACT_TANH) return tanhf(v);
  return v;
}

// One output row = M contiguous floats (M bands of a frame, or M samples of a mono buffer).
__device__ __forceinline__ void store_row(const PqmfParams& p, int s, int row, const float (&y)[M]) {
  float* dst = p.out + static_cast<int64_t>(s) * p.out_sstride + p.out_base + static_cast<int64_t>(row) * M;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {  // (a fused output may be any caller pointer)
    float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < M / 4; ++q) d4[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < M; ++q) dst[q] = y[q];
  }
}

// Sample-major window padded by 4 floats every 32: thread t's aligned float4 at sample 16t+4m
// then falls in a distinct 4-bank group for each of the 8 threads of a quarter warp.
__device__ __forceinline__ int apad(int e) { return e + 4 * (e >> 5); }

// Analysis.  Coefficients ride in the kernel-parameter (constant) bank: uniform across the block,
// they are FFMA operands straight from the constant cache, with no shared-memory traffic.
//   stage 1  u[f][b] = sum_a S[a][b] x[16 f + 32 a + b]: thread (b = lane, 32 frames of warp w);
//            with z[k] = x[16 k + b], u[f] = sum_a S[a][b] z[f + 2 a] — the even and the odd
//            frames are two register-sliding windows (8 taps each): 46 conflict-free loads and
//            256 FMAs per thread, S[.][b] in 8 registers.
//   stage 2  y[f][n] = bias[n] + sum_b Cm[n][b] u[f][b]: thread = frame, u row from shared
//            memory (8 conflict-free 128-bit loads), Cm / bias from the constant bank.
// Same summation order as the plain form (a, then b, ascending).
__global__ void __launch_bounds__(FB) pqmf_analysis_kernel(const PqmfParams p, const __grid_constant__ PqmfCoef k) {
  constexpr int WMAX = M * FB + K - M;
  constexpr int ULD = B + 4;  // u rows: 36 floats, conflict-free 128-bit reads by frame
  __shared__ __align__(16) float win[WMAX];
  __shared__ __align__(16) float us[FB * ULD];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * FB;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float* src = p.in + static_cast<int64_t>(s) * p.in_sstride + p.in_f0 + static_cast<int64_t>(M) * i0;
  const int n_frames = min(FB, p.t_out - i0);
  const int W = M * n_frames + K - M;
  {  // all loads in flight before the first store (the block's only HBM read)
    constexpr int IT = (WMAX + FB - 1) / FB;
    float v[IT];
    if (p.xin) {  // fused mono input: cached rows from the strip, new rows from the caller
      const int a0 = p.in_f0 + M * i0;  // strip row of window element 0
      const float* xs = p.xin + static_cast<int64_t>(s) * p.xin_T - p.cache0;
      float* tail = p.strip + static_cast<int64_t>(s) * p.in_sstride;
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int e = t + it * FB, a = a0 + e;
        v[it] = e < W ? __ldg(a < p.cache0 ? src + e : xs + a) : 0.f;
        if (e < W && a >= p.xin_T) tail[a] = v[it];  // the next call's cache rows
      }
    } else {
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int e = t + it * FB;
        v[it] = e < W ? __ldg(src + e) : 0.f;
      }
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = t + it * FB;
      if (e < WMAX) win[e] = act_apply(v[it], p.pre_act, p.pre_alpha);
    }
  }
  float sb[A];  // S[.][lane]: a per-lane index — from global memory (a lane-divergent constant-bank
                // read would serialise over the 32 addresses)
#pragma unroll
  for (int a = 0; a < A; ++a) sb[a] = __ldg(p.S + a * B + lane);
  __syncthreads();
  {
    const int f0 = warp * 32;
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      float z[16 + A - 1];
#pragma unroll
      for (int m = 0; m < 16 + A - 1; ++m) z[m] = win[M * (f0 + par + 2 * m) + lane];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float u = 0.f;
#pragma unroll
        for (int a = 0; a < A; ++a) u = fmaf(sb[a], z[j + a], u);
        us[(f0 + par + 2 * j) * ULD + lane] = u;
      }
    }
  }
  __syncthreads();
  if (t >= n_frames) return;
  float u[B];
#pragma unroll
  for (int b4 = 0; b4 < B / 4; ++b4) {
    const float4 v = *reinterpret_cast<const float4*>(&us[t * ULD + 4 * b4]);
    u[4 * b4] = v.x, u[4 * b4 + 1] = v.y, u[4 * b4 + 2] = v.z, u[4 * b4 + 3] = v.w;
  }
  float y[M];
#pragma unroll
  for (int n = 0; n < M; ++n) y[n] = k.c[A * B + M * B + n];
#pragma unroll
  for (int b = 0; b < B; ++b) {
#pragma unroll
    for (int n = 0; n < M; ++n) y[n] = fmaf(k.c[A * B + n * B + b], u[b], y[n]);
  }
  if (p.post_act != ACT_ID) {
#pragma unroll
    for (int n = 0; n < M; ++n) y[n] = act_apply(y[n], p.post_act, p.post_alpha);
  }
  store_row(p, s, i0 + t, y);
}

// Synthesis.  Coefficients in the constant bank (see the analysis).
//   stage 1  V[f][c] = sum_ch R[c][ch] x[f][ch] for the NCLS canonical classes: thread = input
//            frame (143 per block: two passes), x row from shared memory, R uniform.
//   stage 2  y[16 i + ph] = bias + sum_q s[q][ph] V[i + q][class(q, ph)]: thread = output row,
//            the MH class values of each (row, q) as 128-bit loads (row stride NCLS + 4: conflict
//            free), s uniform.
template <int P, bool MIR>
__global__ void __launch_bounds__(FB) pqmf_synthesis_kernel(const PqmfParams p, const __grid_constant__ PqmfCoef k) {
  constexpr int MH = MIR ? M / 2 : M;
  constexpr int NCLS = P * MH;
  constexpr int NF = FB + Q - 1;   // input frames per block
  constexpr int XLD = M + 4;       // 20: float4 rows, conflict-free per quarter warp
  constexpr int VLD = NCLS + 4;    // 20 or 36: float4 rows, conflict-free per quarter warp
  __shared__ __align__(16) float xs[NF * XLD];
  __shared__ __align__(16) float V[NF * VLD];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * FB;
  const int t = threadIdx.x;
  const int n_rows = min(FB, p.t_out - i0);
  const int nf = n_rows + Q - 1;
  const float* src = p.in + static_cast<int64_t>(s) * p.in_sstride +
                     (static_cast<int64_t>(p.in_f0) + i0) * p.in_fstride + p.in_off;
  {  // all loads in flight before the first store
    constexpr int IT = (NF * M + FB - 1) / FB;
    float v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = t + it * FB;
      v[it] = e < nf * M ? __ldg(src + static_cast<int64_t>(e / M) * p.in_fstride + e % M) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = t + it * FB;
      if (e < nf * M) xs[(e / M) * XLD + e % M] = act_apply(v[it], p.pre_act, p.pre_alpha);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int f = t; f < nf; f += FB) {
    float x[M];
#pragma unroll
    for (int c4 = 0; c4 < M / 4; ++c4) {
      const float4 v = *reinterpret_cast<const float4*>(&xs[f * XLD + 4 * c4]);
      x[4 * c4] = v.x, x[4 * c4 + 1] = v.y, x[4 * c4 + 2] = v.z, x[4 * c4 + 3] = v.w;
    }
#pragma unroll
    for (int c4 = 0; c4 < NCLS / 4; ++c4) {
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int ch = 0; ch < M; ++ch) acc = fmaf(k.c[(4 * c4 + j) * M + ch], x[ch], acc);
        o[j] = acc;
      }
      *reinterpret_cast<float4*>(&V[f * VLD + 4 * c4]) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();
  if (t >= n_rows) return;
  // prototype: y[ph] = bias + sum_q s[q][ph] V[t + q][class(q, ph)]
  constexpr int SOFF = NCLS * M;
  float y[M];
  const float b0 = k.c[SOFF + Q * M];
#pragma unroll
  for (int ph = 0; ph < M; ++ph) y[ph] = b0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int r = q % P;
    float v[MH];
#pragma unroll
    for (int k4 = 0; k4 < MH / 4; ++k4) {
      const float4 w = *reinterpret_cast<const float4*>(&V[(t + q) * VLD + r * MH + 4 * k4]);
      v[4 * k4] = w.x, v[4 * k4 + 1] = w.y, v[4 * k4 + 2] = w.z, v[4 * k4 + 3] = w.w;
    }
#pragma unroll
    for (int ph = 0; ph < M; ++ph) {
      const int kk = MIR ? (ph < M - 1 - ph ? ph : M - 1 - ph) : ph;
      y[ph] = fmaf(k.c[SOFF + q * M + ph], v[kk], y[ph]);
    }
  }
  if (p.post_act != ACT_ID) {
#pragma unroll
    for (int ph = 0; ph < M; ++ph) y[ph] = act_apply(y[ph], p.post_act, p.post_alpha);
  }
  store_row(p, s, i0 + t, y);
}

}  // namespace

bool pqmf_fast_shape(int kind, int bands, int A_or_Q, int B_or_classes, int period, int mirror) {
  if (bands != M) return false;
  if (kind == 1) return A_or_Q == A && B_or_classes == B;
  return A_or_Q == Q && (period == 1 || period == 2) && B_or_classes == period * (mirror ? M / 2 : M);
}

const void* pqmf_kernel_ptr(int kind, int period, int mirror) {
  if (kind == 1) return reinterpret_cast<const void*>(&pqmf_analysis_kernel);
  if (period == 2)
    return mirror ? reinterpret_cast<const void*>(&pqmf_synthesis_kernel<2, true>)
                  : reinterpret_cast<const void*>(&pqmf_synthesis_kernel<2, false>);
  return mirror ? reinterpret_cast<const void*>(&pqmf_synthesis_kernel<1, true>)
                : reinterpret_cast<const void*>(&pqmf_synthesis_kernel<1, false>);
}

void launch_pqmf(int kind, const PqmfParams& p, const PqmfCoef& k, cudaStream_t st) {
  dim3 grid((p.t_out + FB - 1) / FB, p.streams);
  if (kind == 1) {
    pqmf_analysis_kernel<<<grid, FB, 0, st>>>(p, k);
  } else if (p.period == 2) {
    if (p.mirror)
      pqmf_synthesis_kernel<2, true><<<grid, FB, 0, st>>>(p, k);
    else
      pqmf_synthesis_kernel<2, false><<<grid, FB, 0, st>>>(p, k);
  } else {
    if (p.mirror)
      pqmf_synthesis_kernel<1, true><<<grid, FB, 0, st>>>(p, k);
    else
      pqmf_synthesis_kernel<1, false><<<grid, FB, 0, st>>>(p, k);
  }
}

}  // namespace scb
