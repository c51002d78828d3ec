// Probe: is the FP64 tensor path (mma.sync m8n8k4 f64 -> DMMA) a separate
// pipe from the FP64 FMA pipe on B200? Times DFMA alone, DMMA alone and both
// interleaved in one loop; if "both" finishes in ~max(DFMA, DMMA) time the
// pipes overlap and GEMM-shaped FP64 work (z = P^H y, the S~ rank-1 sums) can
// be moved off the DFMA pipe.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NF, int NM>
__global__ void probe(int iters, double* out, double s) {
  double f[8];
  double acc[4][2];
  double a = threadIdx.x * 1e-3 + s, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = i * s;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < NF; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, a);
#pragma unroll
    for (int r = 0; r < NM; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(acc[i], a, b);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += f[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) t += acc[i][0] + acc[i][1];
  if (t == 12345.678) out[0] = t;
}

template <int NF, int NM>
void run(const char* name, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<NF, NM><<<blocks, threads>>>(iters, out, 0.5);
  cudaEventRecord(e0);
  probe<NF, NM><<<blocks, threads>>>(iters, out, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double dfma_flops = 2.0 * 8 * NF * (double)iters * blocks * threads;
  const double dmma_flops = 512.0 * 4 * NM * (double)iters * warps;
  printf("{\"probe\": \"%s\", \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
         name, ms, dfma_flops / ms / 1e9, dmma_flops / ms / 1e9, (dfma_flops + dmma_flops) / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  run<4, 0>("dfma_only", blocks, threads, iters, out);
  run<0, 1>("dmma_only", blocks, threads, iters, out);
  run<4, 1>("dfma4_dmma1", blocks, threads, iters, out);
  run<2, 1>("dfma2_dmma1", blocks, threads, iters, out);
  run<8, 1>("dfma8_dmma1", blocks, threads, iters, out);
  cudaDeviceSynchronize();
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
