// Legacy warp-level tensor path (mma.sync, SASS HMMA) throughput on sm_100a:
// is it fast enough to carry the pruned kernel's incircle screen (a
// 32 rays x 64 candidates x K=8 tf32 product per warp and tile)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mma_probe.cu -o /tmp/mma_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(32) k_tf32(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

template <int CH>
__global__ void __launch_bounds__(32) k_bf16(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

template <class K>
void run(const char* name, K kern, int ctas, int iters, int ch, double flop_per_mma) {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<ctas, 32>>>(out, iters);
  cudaEventRecord(e0);
  kern<<<ctas, 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)ctas * iters * ch;
  printf("%-28s ctas %6d: %.3f ms, %.1f TFLOP/s, %.2f mma/clk/SM at 1965 MHz\n", name, ctas, ms,
         mmas * flop_per_mma / ms / 1e9, mmas / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}

int main() {
  const int iters = 20000;
  for (int per_sm : {4, 8, 16, 32}) {
    run("tf32 m16n8k8 x4 chains", k_tf32<4>, 148 * per_sm, iters, 4, 2.0 * 16 * 8 * 8);
    run("bf16 m16n8k16 x4 chains", k_bf16<4>, 148 * per_sm, iters, 4, 2.0 * 16 * 8 * 16);
  }
  run("tf32 m16n8k8 x8 chains", k_tf32<8>, 148 * 16, iters, 8, 2.0 * 16 * 8 * 8);
  return 0;
}
