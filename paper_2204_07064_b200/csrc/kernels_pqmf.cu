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

#include "kernels_pqmf.hpp"

namespace scb {

namespace {

constexpr int M = 16;      // bands
constexpr int B = 32;      // 2M modulation phases
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
  if (((p.out_sstride | p.out_base) & 3) == 0) {
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

__global__ void __launch_bounds__(FB) pqmf_analysis_kernel(const PqmfParams p) {
  constexpr int WMAX = M * FB + K - M;
  __shared__ __align__(16) float win[WMAX + 4 * (WMAX / 32 + 1)];
  __shared__ __align__(16) float sS[A * B];
  __shared__ __align__(16) float sC[M * B];
  __shared__ float sb[M];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * FB;
  const int t = threadIdx.x;
  for (int e = t; e < A * B; e += FB) sS[e] = p.S[e];
  for (int e = t; e < M * B; e += FB) sC[e] = p.C[e];
  if (t < M) sb[t] = p.bias[t];
  const float* src = p.in + static_cast<int64_t>(s) * p.in_sstride + p.in_f0 + static_cast<int64_t>(M) * i0;
  const int n_frames = min(FB, p.t_out - i0);
  const int W = M * n_frames + K - M;
  {  // all loads in flight before the first store (the block's only HBM read)
    constexpr int IT = (WMAX + FB - 1) / FB;
    float v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = t + it * FB;
      v[it] = e < W ? __ldg(src + e) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = t + it * FB;
      if (e < W) win[apad(e)] = act_apply(v[it], p.pre_act, p.pre_alpha);
    }
  }
  __syncthreads();
  if (t >= n_frames) return;
  float u[B];
#pragma unroll
  for (int b = 0; b < B; ++b) u[b] = 0.f;
#pragma unroll
  for (int a = 0; a < A; ++a) {
#pragma unroll
    for (int b4 = 0; b4 < B / 4; ++b4) {
      const float4 x = *reinterpret_cast<const float4*>(&win[apad(M * t + B * a + 4 * b4)]);
      const float4 c = *reinterpret_cast<const float4*>(&sS[a * B + 4 * b4]);
      u[4 * b4 + 0] = fmaf(c.x, x.x, u[4 * b4 + 0]);
      u[4 * b4 + 1] = fmaf(c.y, x.y, u[4 * b4 + 1]);
      u[4 * b4 + 2] = fmaf(c.z, x.z, u[4 * b4 + 2]);
      u[4 * b4 + 3] = fmaf(c.w, x.w, u[4 * b4 + 3]);
    }
  }
  float y[M];
#pragma unroll
  for (int n = 0; n < M; ++n) {
    float acc = sb[n];
#pragma unroll
    for (int b4 = 0; b4 < B / 4; ++b4) {
      const float4 c = *reinterpret_cast<const float4*>(&sC[n * B + 4 * b4]);
      acc = fmaf(c.x, u[4 * b4 + 0], acc);
      acc = fmaf(c.y, u[4 * b4 + 1], acc);
      acc = fmaf(c.z, u[4 * b4 + 2], acc);
      acc = fmaf(c.w, u[4 * b4 + 3], acc);
    }
    y[n] = act_apply(acc, p.post_act, p.post_alpha);
  }
  store_row(p, s, i0 + t, y);
}

template <int P, bool MIR>
__global__ void __launch_bounds__(FB) pqmf_synthesis_kernel(const PqmfParams p) {
  constexpr int MH = MIR ? M / 2 : M;
  constexpr int NCLS = P * MH;
  constexpr int NF = FB + Q - 1;   // input frames per block
  constexpr int XLD = M + 4;       // 20: float4 rows, conflict-free per quarter warp
  constexpr int VLD = NCLS + 1;    // odd: conflict-free scalar rows
  __shared__ __align__(16) float xs[NF * XLD];
  __shared__ float V[NF * VLD];
  __shared__ __align__(16) float sR[NCLS * M];
  __shared__ __align__(16) float sv[Q * M];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * FB;
  const int t = threadIdx.x;
  for (int e = t; e < NCLS * M; e += FB) sR[e] = p.C[e];
  for (int e = t; e < Q * M; e += FB) sv[e] = p.S[e];
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
  // modulation: V[f][k] = sum_c R[k][c] x[f][c]; a task is (class group g of 8, frame f), g
  // warp-uniform so the coefficient reads broadcast (and depend on the task: no hoisting)
  constexpr int KG = 8;
  for (int e = t; e < nf * (NCLS / KG); e += FB) {
    const int g = e / nf, f = e - g * nf;
    float x[M];
#pragma unroll
    for (int c4 = 0; c4 < M / 4; ++c4) {
      const float4 v = *reinterpret_cast<const float4*>(&xs[f * XLD + 4 * c4]);
      x[4 * c4] = v.x, x[4 * c4 + 1] = v.y, x[4 * c4 + 2] = v.z, x[4 * c4 + 3] = v.w;
    }
    const float* rg = &sR[g * KG * M];
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      float acc = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < M / 4; ++c4) {
        const float4 r = *reinterpret_cast<const float4*>(&rg[k * M + 4 * c4]);
        acc = fmaf(r.x, x[4 * c4], acc);
        acc = fmaf(r.y, x[4 * c4 + 1], acc);
        acc = fmaf(r.z, x[4 * c4 + 2], acc);
        acc = fmaf(r.w, x[4 * c4 + 3], acc);
      }
      V[f * VLD + g * KG + k] = acc;
    }
  }
  __syncthreads();
  if (t >= n_rows) return;
  // prototype: y[ph] = bias + sum_q s[q][ph] V[t + q][class(q, ph)]
  float y[M];
  const float b0 = p.bias[0];
#pragma unroll
  for (int ph = 0; ph < M; ++ph) y[ph] = b0;
#pragma unroll
  for (int q0 = 0; q0 < Q; q0 += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int q = q0 + r;
      const float* vrow = &V[(t + q) * VLD + r * MH];
      float v[MH];
#pragma unroll
      for (int k = 0; k < MH; ++k) v[k] = vrow[k];
#pragma unroll
      for (int ph4 = 0; ph4 < M / 4; ++ph4) {
        const float4 c = *reinterpret_cast<const float4*>(&sv[q * M + 4 * ph4]);
        const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ph = 4 * ph4 + j;
          const int k = MIR ? (ph < M - 1 - ph ? ph : M - 1 - ph) : ph;
          y[ph] = fmaf(cc[j], v[k], y[ph]);
        }
      }
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

void launch_pqmf(int kind, const PqmfParams& p, cudaStream_t st) {
  dim3 grid((p.t_out + FB - 1) / FB, p.streams);
  if (kind == 1) {
    pqmf_analysis_kernel<<<grid, FB, 0, st>>>(p);
  } else if (p.period == 2) {
    if (p.mirror)
      pqmf_synthesis_kernel<2, true><<<grid, FB, 0, st>>>(p);
    else
      pqmf_synthesis_kernel<2, false><<<grid, FB, 0, st>>>(p);
  } else {
    if (p.mirror)
      pqmf_synthesis_kernel<1, true><<<grid, FB, 0, st>>>(p);
    else
      pqmf_synthesis_kernel<1, false><<<grid, FB, 0, st>>>(p);
  }
}

}  // namespace scb
