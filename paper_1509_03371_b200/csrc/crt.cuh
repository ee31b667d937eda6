// crt.cuh -- the exact conv on the int8 tensor cores by certification (conv_crt.cu): the
// host-side state a net keeps per layer (prepared weights) and per device (scratch).
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace graft {

// Weights prepared once per upload: [15][Mp][k*k][Cp] int8 (14 residue planes + the u8 |w|
// ceilings), per-row exponents and L1 norms, and the fixed-point widths chosen for K.
struct CrtWeights {
  DevBuf planes, ew, w1, nw;
  int M = 0, C = 0, k = 0, bw = 0, bx = 0;
  bool valid = false;
};
// Per-launch scratch (grown on demand): activation residue planes, patch sums, residue /
// bound outputs of the GEMMs, and a small misc block (max|x|, fallback count, overflow list).
struct CrtScratch {
  DevBuf xres, s1, x1, res, sabs, misc, fails, xf, tapoff, approx, s1n, x1n;
  // timed mode: device ms accumulated per stage (0 prep, 1 residue GEMMs, 2 certify, 3 chain)
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  double ms[4] = {0, 0, 0, 0};
  long long gemm_launches = 0;
  // smallest scratch request (bytes) that cudaMalloc refused; requests at least this large go
  // straight to the caller's conv_exact fallback instead of retrying the allocation every call
  size_t refused_bytes = 0;
  ~CrtScratch() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
};

int crt_padded_c(int C);
int crt_num_moduli();
bool conv_crt_eligible(const ConvShape& sh);
void crt_prepare_weights(const float* w_f32, int M, int C, int k, CrtWeights& cw, cudaStream_t st);
size_t crt_scratch_bytes_per_image(const ConvShape& sh);
// Same contract as conv_exact (bit-identical outputs; out / out_relu nullable), for stride-1,
// unpadded layers with K = C*k*k <= 33000. w_f32: [M][C][k][k] f32 (reference order). Returns
// false when uncertified outputs overflowed every list (NaN / Inf operands) or the scratch could
// not be allocated: rerun the layer on conv_exact.
bool conv_crt(const double* in, const CrtWeights& cw, const float* w_f32, const float* bias, const ConvShape& sh,
              double* out, double* out_relu, CrtScratch& scr, cudaStream_t st, bool timed = false);
// Outputs recomputed by the exact chain in the last conv_crt on `scr` (synchronises).
unsigned long long conv_crt_fallbacks(const CrtScratch& scr, cudaStream_t st);

}  // namespace graft
