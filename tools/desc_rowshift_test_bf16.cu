// Experiment (bf16 / SW64 variant): can a K-major SW64 UMMA shared-memory descriptor start at an arbitrary ROW of a
// 1024B-aligned swizzled tile (row offset r = 1..8, i.e. start address not 1024B-aligned)?
// Needed to read several taps of a conv window from ONE swizzled copy of the rows.
// Prints max |err| per (shift, base_offset mode).  Build: nvcc -gencode arch=compute_100a,
// code=sm_100a -o desc_rowshift_test tools/desc_rowshift_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t base_off) {  // SW64 here
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(base_off & 7) << 49;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}
#include <cuda_bf16.h>

constexpr int ROWS = 144, N = 32;

__global__ void k(const float* A, const float* B, float* out, int shift, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(sm);              // ROWS x 32 bf16, SW64
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(sm + ROWS * 64);  // N x 32 bf16, SW64
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int e = t; e < ROWS * 32; e += blockDim.x) {
    const int w = e / 32, c = e % 32;  // chunk = 8 bf16
    sa[w * 32 + (((c >> 3) ^ ((w >> 1) & 3)) << 3) + (c & 7)] = __float2bfloat16(A[e]);
  }
  for (int e = t; e < N * 32; e += blockDim.x) {
    const int w = e / 32, c = e % 32;
    sb[w * 32 + (((c >> 3) ^ ((w >> 1) & 3)) << 3) + (c & 7)] = __float2bfloat16(B[e]);
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t aaddr = smem_u32(sa) + shift * 64 + kk * 32;
      const uint32_t bo = mode == 0 ? 0u : mode == 1 ? ((aaddr >> 7) & 3) : (static_cast<uint32_t>(shift >> 1) & 3);
      const uint64_t da = sw128_desc(aaddr, bo);
      const uint64_t db = sw128_desc(smem_u32(sb) + kk * 32, 0);
      const uint32_t acc = kk > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
      smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tm + ((static_cast<uint32_t>(t / 32) * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) out[t * N + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  std::vector<float> A(ROWS * 32), B(N * 32), out(128 * N);
  for (size_t i = 0; i < A.size(); ++i) A[i] = static_cast<float>((i * 7919) % 97) / 97.f - 0.5f;
  for (size_t i = 0; i < B.size(); ++i) B[i] = static_cast<float>((i * 104729) % 89) / 89.f - 0.5f;
  // tf32 operands: make inputs exactly representable (top 19 bits) so only the shift matters
  for (auto& x : A) x = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, x) & 0xFFFF0000u);
  for (auto& x : B) x = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, x) & 0xFFFF0000u);
  float *dA, *dB, *dO;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dO, out.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + ROWS * 64 + N * 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 3; ++mode) {
    for (int shift = 0; shift <= 9; ++shift) {
      cudaMemset(dO, 0, out.size() * 4);
      k<<<1, 128, smem>>>(dA, dB, dO, shift, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d shift %d: CUDA error %s\n", mode, shift, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int c = 0; c < 32; ++c) ref += static_cast<double>(A[(m + shift) * 32 + c]) * B[n * 32 + c];
          maxerr = std::fmax(maxerr, std::fabs(ref - out[m * N + n]));
        }
      printf("mode %d (%s) shift %d: max|err| = %.3e\n", mode,
             mode == 0 ? "base_off=0" : mode == 1 ? "base_off=(addr>>7)&3" : "base_off=(shift>>1)&3", shift, maxerr);
    }
  }
  return 0;
}
