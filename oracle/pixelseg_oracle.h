/*
 * pixelseg_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 path. It is a plain-C restatement of the
 * reference algorithm (paths relative to /root/reference/proj/include/pixelseg/) and is
 * linked ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the
 * checker -- never by the product library (paper_1509_03371_b200/libgraft_cuda.so).
 *
 * Parity pinned: tests/test_oracle_cpu.py checks every function below against golden
 * vectors produced by the reference itself (oracle/_ref, built from /root/reference by
 * oracle/Makefile, fixtures in tests/golden/ made by tests/golden/make_golden.py) and against
 * the frozen known-answer values of the reference's own tests.
 */
#ifndef PIXELSEG_ORACLE_H
#define PIXELSEG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror include/graft_cuda.h */
#define ORC_OK 0
#define ORC_ESPEC 2
#define ORC_ESIZE 6

const char* orc_last_error(void);

/* ---- Rng: mt19937_64 + hand-rolled transforms (rng.hpp:12-54) ---- */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int have_spare;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n);
double orc_rng_gaussian(orc_rng* r);
double orc_rng_gaussian_ms(orc_rng* r, double mean, double sigma);
/* bulk helpers (one stream, in order) */
void orc_rng_fill_uniform_f32(orc_rng* r, float* dst, size_t n, double lo, double hi);
void orc_rng_fill_uniform_f64(orc_rng* r, double* dst, size_t n, double lo, double hi);
void orc_rng_fill_gaussian_f32(orc_rng* r, float* dst, size_t n, double mean, double sigma);
void orc_rng_fill_gaussian_f64(orc_rng* r, double* dst, size_t n, double mean, double sigma);
void orc_rng_fill_index_u8(orc_rng* r, uint8_t* dst, size_t n, uint64_t m);
size_t orc_rng_state_size(void);

/* ---- ConvGeometry::out_extent (tensor.hpp:26-42) ---- */
int orc_out_extent(int in, int k, int d, int s, int p, const char* what, int* out);

/* ---- im2col_sk (tensor.hpp:80-110); col is (C*k*k) x (oh*ow) ---- */
int orc_im2col_f32(const float* in, int C, int H, int W, int k, int d, int s, int p, float* col);
int orc_im2col_f64(const double* in, int C, int H, int W, int k, int d, int s, int p, double* col);

/* ---- gemm (tensor.hpp:151-169): fp64 accumulator, ascending kk ---- */
void orc_gemm_f32(int ta, int tb, int m, int n, int k, float alpha, const float* a, const float* b,
                  float beta, float* c);
void orc_gemm_f64(int ta, int tb, int m, int n, int k, double alpha, const double* a,
                  const double* b, double beta, double* c);

/* ---- conv_sk_forward (layers.hpp:43-64) as the direct loop of oracles.hpp:51-82 ---- */
int orc_conv_f32(const float* in, int C, int H, int W, const float* w, const float* b, int f_out,
                 int k, int d, int s, int p, float* out);
int orc_conv_f64(const double* in, int C, int H, int W, const double* w, const double* b,
                 int f_out, int k, int d, int s, int p, double* out);
/* same, split over nthreads (pthreads) by output channel; bit-identical */
int orc_conv_f32_mt(const float* in, int C, int H, int W, const float* w, const float* b, int f_out,
                    int k, int d, int s, int p, float* out, int nthreads);

/* ---- maxpool_sk_forward (layers.hpp:102-132); argmax may be NULL ---- */
int orc_maxpool_f32(const float* in, int C, int H, int W, int k, int d, int s, float* out,
                    uint64_t* argmax);
int orc_maxpool_f64(const double* in, int C, int H, int W, int k, int d, int s, double* out,
                    uint64_t* argmax);

/* ---- relu / upconv / mergecrop / softmax (layers.hpp:143-147,162-176,196-212,227-244) ---- */
void orc_relu_f32(const float* in, size_t n, float* out);
void orc_relu_f64(const double* in, size_t n, double* out);
void orc_upconv_f32(const float* in, int C, int H, int W, float* out);
void orc_upconv_f64(const double* in, int C, int H, int W, double* out);
int orc_mergecrop_f32(const float* a, int Ca, int Ha, int Wa, const float* b, int Cb, int Hb,
                      int Wb, float* out);
int orc_mergecrop_f64(const double* a, int Ca, int Ha, int Wa, const double* b, int Cb, int Hb,
                      int Wb, double* out);
void orc_softmax_f32(const float* in, int C, int H, int W, float* out);
void orc_softmax_f64(const double* in, int C, int H, int W, double* out);

/* ---- preprocessing (pipeline.hpp:36-58, 86-93) ---- */
int orc_mirror_pad_u8(const uint8_t* img, int H, int W, int v, uint8_t* out);
void orc_normalize_f32(const uint8_t* img, size_t n, float* out);
void orc_normalize_f64(const uint8_t* img, size_t n, double* out);

/* ---- process() tile helpers (pipeline.hpp:662-694) ---- */
/* number of tile offsets along an extent, and the offsets themselves */
int orc_tile_offsets(int extent, int w, int* offs, int cap);
/* per-pixel argmax (strict '>', first wins) + stitch of one tile's probabilities */
void orc_stitch_f32(const float* tile_probs, int C, int w, int oy, int ox, int H, int W,
                    uint8_t* labels, float* probs);

/* ---- MALIS (malis.hpp) ---- */
void orc_affinity_forward_f32(const float* img, int h, int w, float* ax, float* ay, uint8_t* mx, uint8_t* my);
void orc_affinity_forward_f64(const double* img, int h, int w, double* ax, double* ay, uint8_t* mx, uint8_t* my);
void orc_affinity_backward_f32(const float* dax, const float* day, const uint8_t* mx, const uint8_t* my, int h,
                               int w, float* dpos, float* dneg);
void orc_affinity_backward_f64(const double* dax, const double* day, const uint8_t* mx, const uint8_t* my, int h,
                               int w, double* dpos, double* dneg);
void orc_connected_components(const uint8_t* lab, int h, int w, int* comp);
void orc_malis_gradient_f32(const float* pax, const float* pay, const float* tax, const float* tay,
                            const int* comp, int h, int w, float* dax, float* day, long long* posx,
                            long long* posy, long long* negx, long long* negy, long long* totals,
                            double* losses);
void orc_malis_gradient_f64(const double* pax, const double* pay, const double* tax, const double* tay,
                            const int* comp, int h, int w, double* dax, double* day, long long* posx,
                            long long* posy, long long* negx, long long* negy, long long* totals,
                            double* losses);
int orc_malis_softmax_loss_f32(const float* scores, int C, int h, int w, const uint8_t* fg, float* diff,
                               double* loss);
int orc_malis_softmax_loss_f64(const double* scores, int C, int h, int w, const uint8_t* fg, double* diff,
                               double* loss);

#ifdef __cplusplus
}
#endif
#endif
