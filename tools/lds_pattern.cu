// Shared-memory wavefronts of row-per-lane loads from a 128-byte-row, 128B-swizzled tile (the 3xFP16
// transform's access pattern, kernels_tc.cu) under different lane -> address mappings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/lds_pattern tools/lds_pattern.cu
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum tools/bin/lds_pattern
#include <cstdio>
#include <cuda_runtime.h>

template <int P> __global__ void k(float* out, int iters) {
  __shared__ __align__(1024) float tile[128 * 32];
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) tile[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = w * 32 + l;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (P == 0) {  // row per lane, chunk j ^ (r & 7): the transform's pattern
        const float4 v = reinterpret_cast<const float4*>(tile)[r * 8 + (j ^ (r & 7))];
        acc += v.x + v.y + v.z + v.w;
      } else if (P == 1) {  // 8 lanes read one row's 8 chunks (contiguous 128 B)
        const int row = w * 32 + (l >> 3) + 4 * j;
        const float4 v = reinterpret_cast<const float4*>(tile)[row * 8 + (l & 7)];
        acc += v.x + v.y + v.z + v.w;
      } else if (P == 2) {  // row per lane, 64-bit loads, lanes l and l + 8 take opposite halves
        const int h = (l >> 3) & 1;
        const float2 a = reinterpret_cast<const float2*>(tile)[r * 16 + 2 * (j ^ (r & 7)) + h];
        const float2 b = reinterpret_cast<const float2*>(tile)[r * 16 + 2 * (j ^ (r & 7)) + (h ^ 1)];
        acc += a.x + a.y + b.x + b.y;
      } else if (P == 3) {  // row per lane, lanes l + 8 start four chunks further
        const float4 v = reinterpret_cast<const float4*>(tile)[r * 8 + ((j ^ (r & 7)) ^ (((l >> 3) & 1) << 2))];
        acc += v.x + v.y + v.z + v.w;
      } else if (P == 4) {  // row per lane, no swizzle (8-way conflict reference)
        const float4 v = reinterpret_cast<const float4*>(tile)[r * 8 + j];
        acc += v.x + v.y + v.z + v.w;
      } else {  // row per lane, 64-bit loads, plain
        const float2 a = reinterpret_cast<const float2*>(tile)[r * 16 + 2 * (j ^ (r & 7))];
        const float2 b = reinterpret_cast<const float2*>(tile)[r * 16 + 2 * (j ^ (r & 7)) + 1];
        acc += a.x + a.y + b.x + b.y;
      }
    }
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int P> void run(float* d, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  k<P><<<148, 128>>>(d, 10);
  cudaEventRecord(a);
  k<P><<<148, 128>>>(d, 20000);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-60s %8.3f ms\n", name, ms);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 128 * 4);
  run<0>(d, "P0 LDS.128 row/lane, chunk j^(r&7) [transform]");
  run<1>(d, "P1 LDS.128 8 lanes = one row (contiguous)");
  run<2>(d, "P2 LDS.64 row/lane, lanes l, l+8 opposite halves");
  run<3>(d, "P3 LDS.128 row/lane, lanes l+8 shifted 4 chunks");
  run<4>(d, "P4 LDS.128 row/lane, unswizzled (conflict reference)");
  run<5>(d, "P5 LDS.64 row/lane, plain halves");
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
