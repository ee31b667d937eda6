// Micro-probes of the DMMA issue rate with conv_exact's operand patterns (no global memory):
// how close can a TM x TN warp tile with per-k-group LDS fragment loads get to the pure-DMMA
// peak?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_probe2 tools/dmma_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int TM, int TN, bool LDS, int MINB>
__global__ void __launch_bounds__(256, MINB) probe(double* out, int iters) {
  __shared__ double s[2][16][32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2 * 16 * 32; i += blockDim.x) (&s[0][0][0])[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double acc[TM][TN][2];
#pragma unroll
  for (int j = 0; j < TM; ++j)
#pragma unroll
    for (int i = 0; i < TN; ++i) acc[j][i][0] = acc[j][i][1] = j + i;
  double af[TM], bf[TN];
#pragma unroll
  for (int j = 0; j < TM; ++j) af[j] = s[0][j][lane];
#pragma unroll
  for (int i = 0; i < TN; ++i) bf[i] = s[1][i][lane];
  for (int it = 0; it < iters; ++it) {
    if (LDS) {
#pragma unroll
      for (int i = 0; i < TN; ++i) bf[i] = s[1][(i + it) & 15][lane];
    }
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      if (LDS) af[j] = s[0][(j + it) & 15][lane];
#pragma unroll
      for (int i = 0; i < TN; ++i) dmma(acc[j][i][0], acc[j][i][1], af[j], bf[i]);
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < TM; ++j)
#pragma unroll
    for (int i = 0; i < TN; ++i) t += acc[j][i][0] + acc[j][i][1];
  if (t == 1.2345) out[0] = t;
}

template <int TM, int TN, bool LDS, int MINB>
void run(const char* name, double* d, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000 / (TM * TN / 16 + 1);
  probe<TM, TN, LDS, MINB><<<sms * MINB, 256>>>(d, 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<TM, TN, LDS, MINB><<<sms * MINB, 256>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double fl = 2.0 * 256 * TM * TN * (double)iters * 8 * sms * MINB;
  printf("%-34s %.2f TFLOP/s\n", name, fl / best * 1e-9);
}

int main() {
  double* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 4, false, 1>("8x4 regs only, 1 CTA", d, sms);
  run<8, 4, true, 1>("8x4 + LDS frags, 1 CTA", d, sms);
  run<4, 4, false, 2>("4x4 regs only, 2 CTA", d, sms);
  run<4, 4, true, 2>("4x4 + LDS frags, 2 CTA", d, sms);
  run<4, 2, false, 3>("4x2 regs only, 3 CTA", d, sms);
  run<4, 2, true, 3>("4x2 + LDS frags, 3 CTA", d, sms);
  run<2, 2, false, 4>("2x2 regs only, 4 CTA", d, sms);
  run<4, 4, false, 1>("4x4 regs only, 1 CTA", d, sms);
  run<2, 4, true, 3>("2x4 + LDS frags, 3 CTA", d, sms);
  return 0;
}
