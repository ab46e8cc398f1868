// Microbenchmark: issue throughput of the transform's instruction mix on sm_100a (cycles per warp
// instruction per SM sub-partition), 4 warps per SMSP, 8 independent chains per thread.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; u[i] = threadIdx.x + i * 77; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { __half2 h = __floats2half2_rn(a[i], a[(i + 1) & 7]); u[i] ^= *reinterpret_cast<uint32_t*>(&h); a[i] += 1.0f; }
      if (OP == 1) { __half2 h = *reinterpret_cast<__half2*>(&u[i]); float2 f = __half22float2(h); a[i] += f.x; u[i] += 3; }
      if (OP == 2) { unsigned long long r, x; float2 v = make_float2(a[i], a[(i+1)&7]); x = *reinterpret_cast<unsigned long long*>(&v);
                     asm volatile("add.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(x)); float2 w = *reinterpret_cast<float2*>(&r); a[i] = w.x - w.y; }
      if (OP == 3) { a[i] = a[i] * 1.0001f; }
      if (OP == 4) { u[i] = (u[i] + 0x1000u) & 0xFFFFE000u; u[i] += 7; }
      if (OP == 5) { a[i] = fmaxf(a[i], a[(i + 3) & 7] * 0.5f); }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 512 * 4); cudaMallocManaged(&cyc, 8);
  const char* names[] = {"F2FP pack (+xor,+fadd)", "HADD2.F32 unpack (+fadd,+iadd)", "FADD2 (+fadd)", "FMUL", "IADD+LOP (+iadd)", "FMUL+FMNMX"};
  const int iters = 4096;
  for (int op = 0; op < 6; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) { case 0: k<0><<<148, 512>>>(out, iters, cyc); break; case 1: k<1><<<148, 512>>>(out, iters, cyc); break;
        case 2: k<2><<<148, 512>>>(out, iters, cyc); break; case 3: k<3><<<148, 512>>>(out, iters, cyc); break;
        case 4: k<4><<<148, 512>>>(out, iters, cyc); break; default: k<5><<<148, 512>>>(out, iters, cyc); }
      cudaDeviceSynchronize();
    }
    // 16 warps per SM = 4 per SMSP; per SMSP instructions-groups = 4 warps * iters * 8
    printf("%-34s %.2f cycles per warp-op-group per SMSP\n", names[op], (double)*cyc / (4.0 * iters * 8));
  }
  return 0;
}
