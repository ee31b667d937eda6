// Minimal TMA box-load probe (debugging conv_tma). Usage: tma_probe <variant>
//  0: 4-D f64 param desc, x=-3   1: x=0   2: 2-D f64   3: 4-D f32   4: desc in global memory
//  5: 2-D f32 x=0 (most basic)   6: 4-D f64 x=0, L2 promotion none
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int RANK>
__device__ void load(uint64_t desc, void* buf, uint64_t* bar, int x, int y, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(bar)), "r"(bytes) : "memory");
  if (RANK == 4)
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                 ::"r"(su(buf)), "l"(desc), "r"(x), "r"(y), "r"(0), "r"(0), "r"(su(bar)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(su(buf)), "l"(desc), "r"(x), "r"(y), "r"(su(bar)) : "memory");
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(bar)) : "memory");
}

template <int RANK>
__global__ void k_param(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, double* out, int x, int y, unsigned bytes) {
  __shared__ __align__(1024) double buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t desc = gtm ? (uint64_t)gtm : (uint64_t)&tm;
    load<RANK>(desc, buf, &bar, x, y, bytes);
    for (int i = 0; i < 32; ++i) out[i] = buf[i];
  }
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  const int W = 40, H = 10;
  std::vector<double> h(W * H * 2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o; cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 64 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  alignas(64) CUtensorMap tm;
  const bool f32 = (v == 3 || v == 5);
  const int es = f32 ? 4 : 8;
  const int rank = (v == 2 || v == 5) ? 2 : 4;
  cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, 2, 1};
  cuuint64_t str[3] = {(cuuint64_t)W * es, (cuuint64_t)W * es * H, (cuuint64_t)W * es * H * 2};
  cuuint32_t box[4] = {16, 2, 1, 1};
  cuuint32_t est[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, d, dims, str, box, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   v == 6 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gtm = nullptr;
  if (v == 4) { cudaMalloc(&gtm, sizeof tm); cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice); }
  const int x = argc > 2 ? atoi(argv[2]) : ((v == 0) ? -3 : 0);
  const unsigned bytes = 16 * 2 * es;
  if (rank == 4) k_param<4><<<1, 32>>>(tm, gtm, o, x, 1, bytes);
  else k_param<2><<<1, 32>>>(tm, gtm, o, x, 1, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d x=%d encode=%d kernel=%s\n", v, x, (int)r, cudaGetErrorString(e));
  return e != cudaSuccess;
}
