// FP64 peak probe for B200 (sm_100a): register-only DMMA (mma.sync f64) and DFMA chains.
// Measures FLOP/s with CUDA events and the SM clock seen by the kernel (clock64 vs %globaltimer).
// Used once to pin the FP64 tensor-core denominator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int NACC>
__global__ void dmma884(double* out, int iters, unsigned long long* clk) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  uint64_t t0 = clock64(), g0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  uint64_t t1 = clock64(), g1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = g1 - g0; }
}

template <int NACC>
__global__ void dmma16816(double* out, int iters, unsigned long long* clk) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  uint64_t t0 = clock64(), g0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  uint64_t t1 = clock64(), g1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = g1 - g0; }
}

template <int NACC>
__global__ void dfma(double* out, int iters, unsigned long long* clk) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  uint64_t t0 = clock64(), g0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  uint64_t t1 = clock64(), g1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = g1 - g0; }
}

typedef void (*kfn)(double*, int, unsigned long long*);

static void run(const char* name, kfn k, int blocks, int threads, int iters, double flop_per_thread_iter) {
  double* out; unsigned long long* clk;
  cudaMalloc(&out, 8); cudaMallocManaged(&clk, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, iters / 10, clk);
  cudaDeviceSynchronize();
  float best = 1e30f; double mhz = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) { best = ms; mhz = (double)clk[0] / (double)clk[1] * 1e3; }
  }
  double flops = flop_per_thread_iter * (double)threads * blocks * iters;
  printf("{\"probe\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.3f, \"sm_mhz_kernel\": %.0f, \"err\": \"%s\"}\n",
         name, blocks, threads, best, flops / best / 1e9, mhz, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(clk);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  int sm = p.multiProcessorCount;
  // m8n8k4: 8*8*4 FMA = 256 FMA = 512 flop per warp-instruction -> 16 flop per thread per mma
  for (int w : {4, 8, 16}) {
    run("dmma_m8n8k4_acc4", dmma884<4>, sm, 32 * w, 200000, 16.0 * 4);
    run("dmma_m8n8k4_acc8", dmma884<8>, sm, 32 * w, 100000, 16.0 * 8);
  }
  run("dmma_m8n8k4_acc8_2x", dmma884<8>, 2 * sm, 256, 100000, 16.0 * 8);
  // m16n8k16: 16*8*16 = 2048 FMA = 4096 flop per warp -> 128 flop/thread
  for (int w : {4, 8}) run("dmma_m16n8k16_acc4", dmma16816<4>, sm, 32 * w, 25000, 128.0 * 4);
  for (int w : {8, 16, 32}) run("dfma_acc8", dfma<8>, sm, 32 * w, 100000, 2.0 * 8);
  run("dfma_acc8_4x", dfma<8>, 4 * sm, 256, 100000, 2.0 * 8);
  return 0;
}
