// Are the FP64 tensor path (DMMA) and the FP64 FMA path (DFMA) separate pipes on B200? If they
// were, an exact conv could split its chains between them. Each CTA runs `dmma_warps` warps of
// back-to-back DMMA.8x8x4 and `dfma_warps` warps of independent DFMA chains; compare the
// combined FLOP rate with each alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_pipes_probe tools/fp64_pipes_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(512, 1) probe(double* out, int iters, int dmma_warps, int dfma_warps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double t = 0;
  if (warp < dmma_warps) {
    double acc[16][2];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = j;
    const double a = 1.0 + lane * 1e-9, b = 1.0 - lane * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dmma(acc[j][0], acc[j][1], a, b);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) t += acc[j][0] + acc[j][1];
  } else if (warp < dmma_warps + dfma_warps) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = j;
    const double a = 1.0 + lane * 1e-9, b = 1.0 - lane * 1e-9;
    for (int it = 0; it < iters; ++it) {
      // 16 independent chains, 16 DFMA per chain per iteration = the DMMA warps' FMA count
      // per iteration would be 16 DMMA x 256 FMA / 32 lanes = 128 per lane; match the time
      // base instead: report FLOPs separately below.
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma(a, acc[j], b);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) t += acc[j];
  }
  if (t == 1.2345) out[0] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  const int cfg[][2] = {{8, 0}, {16, 0}, {0, 8}, {0, 16}, {8, 8}, {4, 12}, {12, 4}};  // <= 16 warps
  for (const auto& c : cfg) {
    probe<<<sms, 512>>>(d, 10, c[0], c[1]);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      probe<<<sms, 512>>>(d, iters, c[0], c[1]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // DMMA: 16 per iteration per warp, 512 FLOP each; DFMA: 8*16 per iteration per lane, 2 FLOP
    const double fl_dmma = static_cast<double>(sms) * c[0] * iters * 16 * 512;
    const double fl_dfma = static_cast<double>(sms) * c[1] * 32 * iters * 128 * 2;
    printf("dmma_warps %2d dfma_warps %2d: %8.3f ms  DMMA %6.2f TF  DFMA %6.2f TF  total %6.2f TF\n", c[0],
           c[1], best, fl_dmma / best / 1e9, fl_dfma / best / 1e9, (fl_dmma + fl_dfma) / best / 1e9);
  }
  return 0;
}
