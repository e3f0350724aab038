#include <cstdio>
#include <cuda_runtime.h>
// DFMA peak: 8 independent chains per thread
__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void dmma_peak(double* out, int iters, double a, double b) {
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double aa = a + threadIdx.x * 1e-9, bb = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i], aa, bb);
  }
  double s = 0; for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__device__ __forceinline__ void dmma16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
template <int NACC>
__global__ void dmma16_peak(double* out, int iters, double a, double b) {
  double c[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double av[8], bv[4];
  for (int j = 0; j < 8; ++j) av[j] = a + j * 1e-9 + threadIdx.x * 1e-12;
  for (int j = 0; j < 4; ++j) bv[j] = b + j * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma16(c[i], av, bv);
  }
  double s = 0; for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
template <typename K>
void run(const char* name, K kern, int blocks, int threads, int iters, double flop_per_thread_iter) {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = double(blocks) * threads * iters * flop_per_thread_iter * reps;
  printf("%-24s blocks=%5d threads=%4d  %8.3f ms  %7.2f TFLOP/s  err=%s\n", name, blocks, threads, ms / reps,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  for (int bps : {1, 2, 4, 8})
    run("dfma", dfma_peak, sms * bps, 256, 20000, 16.0);
  for (int bps : {1, 2, 4})
    run("dmma m8n8k4 x8", dmma_peak<8>, sms * bps, 256, 10000, 256.0 * 2 * 8 / 32);
  for (int bps : {1, 2, 4})
    run("dmma m8n8k4 x16", dmma_peak<16>, sms * bps, 256, 5000, 256.0 * 2 * 16 / 32);
  for (int bps : {1, 2, 4})
    run("dmma m16n8k16 x4", dmma16_peak<4>, sms * bps, 256, 2000, 16.0*8*16 * 2 * 4 / 32);
  return 0;
}
