// tf32_peak.cu — measured tensor-core peak of tcgen05 kind::tf32 (and kind::f16 bf16 as the
// methodology check against MEASURED_PEAKS.json's cuBLAS bf16 figure) on this B200.
//
// One persistent CTA per SM; the operand tiles (random tf32 / bf16 values — data-dependent
// power is part of the peak) stay resident, one elected lane of warp 0 issues `iters` x (K-row
// of 4 MMAs) of M128 x N x K into a TMEM accumulator:
//   mode 0: SS  kind::tf32  (A and B from 128B-swizzled shared memory), K = 8 per MMA
//   mode 1: TS  kind::tf32  (A from TMEM, B from shared memory)   — the form conv_tc_kernel uses
//   mode 2: SS  kind::f16 with bf16 operands, K = 16 per MMA
//   mode 3: TS  kind::f16 with fp16 operands (A from TMEM), K = 16 per MMA — the 3xFP16 path
// FLOPs per MMA = 2 x 128 x N x K.  Driven by tools/tf32_peak.py (ctypes; CUDA events; burst =
// one ~20 ms launch, sustained = back-to-back launches for 4 s; NVML clocks sampled alongside).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o tools/bin/libtf32_peak.so tools/tf32_peak.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void mma_ss(int mode, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  if (mode == 2) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}

__device__ __forceinline__ void mma_ts_f16(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ float rnd(uint32_t i) {
  return (static_cast<float>(hash(i) >> 8) * (1.0f / 8388608.0f)) - 1.0f;  // [-1, 1)
}

template <int mode>
__global__ void __launch_bounds__(128, 1) peak_kernel(int n, int iters, float* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sa = sm;                  // 128 rows x 128 B
  uint8_t* sb = sm + 128 * 128;      // n rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // operands: random values (tf32: fp32 bit patterns; bf16: packed pairs); the swizzle only
  // permutes 16-byte chunks within a row, irrelevant for random data
  for (int i = tid; i < (128 + n) * 32; i += blockDim.x) {
    const float v = rnd(i * 2654435761u + blockIdx.x);
    if (mode == 3) {
      const __half2 h2 = __floats2half2_rn(v, rnd(i + 77777u));
      reinterpret_cast<__half2*>(sm)[i] = h2;
    } else if (mode == 2) {
      uint32_t lo = __float_as_uint(v) >> 16, hi = __float_as_uint(rnd(i + 77777u)) >> 16;
      reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
    } else {
      reinterpret_cast<float*>(sm)[i] = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp-uniform (shfl) so the MMA operands live in uniform registers: no R2UR waterfall
  const uint32_t tbase = __shfl_sync(0xffffffffu, tslot, 0);
  if (mode == 1 || mode == 3) {
    // A (128 x 32 tf32 / 128 x 64 fp16) into TMEM columns [256, 288): lane = row, warp w owns lanes 32w..
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = rnd((tid * 32 + j) * 2246822519u + 13u);
    const uint32_t ta = tbase + (static_cast<uint32_t>(warp * 32) << 16) + 256;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const uint32_t fmt = mode == 2 ? 1u : mode == 3 ? 0u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                           (static_cast<uint32_t>(128 >> 4) << 24);
    const uint64_t ad = sw128_desc(__shfl_sync(0xffffffffu, smem_u32(sa), 0));
    const uint64_t bd = sw128_desc(__shfl_sync(0xffffffffu, smem_u32(sb), 0));
    // the accumulator ping-pongs between columns [0, n) and [n, 2n) when 2n <= 256
    const uint32_t dstep = (2 * n <= 256) ? static_cast<uint32_t>(n) : 0u;
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tbase + ((it & 1) ? dstep : 0u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (it > 1 || kk > 0) ? 1u : 0u;
        if (mode == 1)
          mma_ts(d, tbase + 256 + kk * 8, bd + 2 * kk, idesc, acc);   // +32 B = +2 in the address field
        else if (mode == 3)
          mma_ts_f16(d, tbase + 256 + kk * 8, bd + 2 * kk, idesc, acc);
        else
          mma_ss(mode, d, ad + 2 * kk, bd + 2 * kk, idesc, acc);
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // read one accumulator value so the work is observable
  if (warp == 0) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tbase) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (tid == 0) sink[blockIdx.x] = __uint_as_float(r);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

}  // namespace

extern "C" {

// Launch `launches` back-to-back kernels on `blocks` CTAs; returns device ms (CUDA events) or
// a negative CUDA error code.
float tf32_peak_run(int mode, int n, int iters, int blocks, int launches) {
  const size_t smem = 1024 + static_cast<size_t>(128 + n) * 128;
  auto kern = mode == 0 ? peak_kernel<0> : mode == 1 ? peak_kernel<1> : mode == 2 ? peak_kernel<2> : peak_kernel<3>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  float* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(float) * blocks) != cudaSuccess) return -1.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 128, smem>>>(n, 8, sink);  // warm (module load, TMEM)
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int l = 0; l < launches; ++l) kern<<<blocks, 128, smem>>>(n, iters, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (err == cudaSuccess) err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return err == cudaSuccess ? ms : -static_cast<float>(err);
}

}  // extern "C"
