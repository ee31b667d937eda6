// kernels.cuh -- launchers of the sm_100a kernels (one per reference hot-path function).
// Activations on the device are stored as f64 holding float values exactly ("widened f32"):
// the conv's DMMA operands need no per-use conversion, and every non-conv layer's result is
// still the reference's float result, bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace graft {

// Shape of one conv_sk launch over a batch of B images (tiles) of C x H x W.
struct ConvShape {
  int B = 1, C = 0, H = 0, W = 0;  // input
  int M = 0;                       // f_out
  int k = 1, d = 1, s = 1, p = 0;
  int OH = 0, OW = 0;
  int in_wp = 0, out_wp = 0;       // row pitches in doubles (0 = compact)
};

// ---- conv_exact.cu ------------------------------------------------------------------------
// Device layout of conv weights for the DMMA kernel: f64, K padded to 16 taps, M padded to
// the 128-row block, tiled as [M/128][K/4][16][32] so one 16-tap chunk of one 128-row block
// is one contiguous 16 KB run in DMMA A-fragment order (lane = m_local*4 + k_local).
size_t conv_weight_tiled_elems(int M, int K);
void tile_conv_weights(const float* w_f32_dev, int M, int K, double* tiled, cudaStream_t st);

// out[b][m][oy][ox] = float(sum_kk w[m][kk]*x[b][kk-tap]) + bias[m], the sum an fp64 fma chain
// in ascending kk (bit-identical to conv_sk_forward, layers.hpp:43-64). Outputs are nullable:
// out_f64 = conv blob, out_relu_f64 = relu(conv) (fused relu_forward), out_f32 = conv as f32.
void conv_exact(const double* in, const double* w_tiled, const float* bias, const ConvShape& sh,
                double* out_f64, double* out_relu_f64, float* out_f32, cudaStream_t st);
// The same for 1x1 convs with f_out <= 8 (two-class heads), from the f32 weights [M][C]: one
// thread per pixel, the f_out chains in registers (conv_exact.cu conv_narrow_kernel).
bool conv_narrow_eligible(const ConvShape& sh);
void conv_narrow(const double* in, const float* w_f32, const float* bias, const ConvShape& sh, double* out_f64,
                 double* out_relu_f64, float* out_f32, cudaStream_t st);

// TMA-fed variant (conv_tma.cu) used by conv_exact for stride-1 layers with 16-byte row
// pitches (every net blob); same arithmetic, same results.
bool conv_tma_eligible(const ConvShape& sh);
void conv_tma(const double* in, const double* w_tiled, const float* bias, const ConvShape& sh,
              double* out_f64, double* out_relu_f64, float* out_f32, cudaStream_t st);

// S=double variant (tests / LayerState<double>): products rounded, mul then add, no FMA,
// exactly like the reference's x86-64 build. Weights f64 row-major [M][K].
void conv_f64_muladd(const double* in, const double* w, const double* bias, const ConvShape& sh,
                     double* out, cudaStream_t st);

// ---- conv_tc.cu (tolerance mode, opt-in) ---------------------------------------------------
// tcgen05 implicit-GEMM conv: bf16 (kind::f16) or tf32 (kind::tf32) operands, f32 accumulation
// in TMEM. NOT bit-exact; see conv_tc.cu and DESIGN.md "Tolerance mode".
enum { TC_BF16 = 1, TC_TF32 = 2, TC_BF16X3 = 3 };
struct TcShape {
  int B = 1, C = 0, H = 0, W = 0;  // input, NHWC per image
  int M = 0, k = 1, d = 1, s = 1, p = 0;
  int OH = 0, OW = 0;
  int out_wp = 0;                  // output row pitch (elements; 0 = OW)
};
int tc_block_k(int kind);
size_t tc_elem_bytes(int kind);
int tc_planes(int kind);  // 2 for the split kinds (hi plane, then lo plane), else 1
// Operand layouts pad channels to the 128-byte K block and f_out to the 128-row MMA tile
// with zeros: [Mp][k][k][Cp] weights, [B][H][W][Cp] activations.
int tc_padded_c(int kind, int C);
int tc_padded_m(int M);
size_t tc_weight_bytes(int kind, int M, int C, int k);
size_t tc_input_bytes(int kind, int B, int C, int H, int W);
bool conv_tc_eligible(int kind, const TcShape& sh);
void weights_to_tc(int kind, const float* w, int M, int C, int k, void* out, cudaStream_t st);
template <typename S>
void chw_to_nhwc(int kind, const S* in, int B, int C, int H, int W, int wp, void* out, cudaStream_t st);
// maxpool_sk_forward on the tensor-core operand layout (in/out [planes][B][H][W][Cp]).
void maxpool_tc(int kind, const void* in, int B, int C, int H, int W, int k, int d, int s, int OH, int OW,
                void* out, cudaStream_t st);
// out (f32, or f64 widened f32 when out_f64) = conv + bias (relu'd when relu); out_relu
// (f64 only, nullable) = relu(conv + bias). CHW per image, row pitch sh.out_wp. out_nhwc
// (nullable): relu(conv + bias) written directly as the next tensor-core conv's operand,
// [B][OH][OW][tc_padded_c(kind, M)] (the padding channels are left untouched: zero them once).
void conv_tc(int kind, const void* x_nhwc, const void* w_tc, const float* bias, const TcShape& sh,
             void* out, void* out_relu, bool out_f64, bool relu, cudaStream_t st,
             void* out_nhwc = nullptr);

// ---- train.cu: the backward layer functions and sgd_step (bit-identical, S = float) --------
// Data blobs: widened-f32 f64, row pitch wp; diffs: compact f32 [C][H][W] of one image.
// gemm (tensor.hpp:151-169) on DMMA: C(i,j) = float(alpha*chain + beta*C), f64 operands
// (float values), 4-stage cp.async pipeline, CTA tile chosen by shape. a_k_contig: A(i,kk) = a[i*lda + kk], else a[kk*lda + i]; likewise B
// with B(kk,j) = b[j*ldb + kk] (k contiguous) or b[kk*ldb + j].
void gemm_dmma_f64ops(int m, int n, int k, const double* a, bool a_k_contig, long long lda,
                      const double* b, bool b_k_contig, long long ldb, double alpha, double beta,
                      float* c, cudaStream_t st);
void widen_f32(const float* in, long long n, double* out, cudaStream_t st);
void transpose_f32(const float* in, int rows, int cols, float* out, cudaStream_t st);
struct DevBuf;
// conv_sk_backward's W^T * dOut (gemm TN) on the forward conv kernel as a 1x1 convolution;
// dy64 = dOut widened, compact [f_out][OH*OW]; col_grad f32 [fan_in][OH*OW]. Scratch buffers
// (transposed / tiled weights, zero bias) are grown as needed.
void col_grad_conv(const double* dy64, int f_out, int OH, int OW, const float* w_f32, int fan_in,
                   DevBuf& wt_f32, DevBuf& wt_tiled, DevBuf& zero_bias, float* col_grad, cudaStream_t st);
void im2col_pitched(const double* in, int C, int H, int W, int wp, int k, int d, int s, int p,
                    int OH, int OW, double* col, cudaStream_t st);
void bias_grad(const float* dout, int M, int n, float* bdiff, cudaStream_t st);
void col2im_add(const float* colg, int C, int H, int W, int k, int d, int s, int p, int OH, int OW,
                float* diff, cudaStream_t st);
void maxpool_backward(const uint64_t* argmax, const float* dout, int C, int H, int W, int k, int d,
                      int s, int OH, int OW, float* din, cudaStream_t st);
// API form: any argmax table (indices outside their window fall back to the reference's
// serial scatter; indices outside the input throw SizeError).
void maxpool_backward_checked(const uint64_t* argmax, const float* dout, int C, int H, int W, int k,
                              int d, int s, int OH, int OW, float* din, size_t n_in, cudaStream_t st);
void maxpool_backward_scatter(const uint64_t* argmax, const float* dout, long long n_out, float* din,
                             size_t n_in, cudaStream_t st);
void relu_backward(const double* data, int rows, int W, int wp, const float* dout, float* din,
                   cudaStream_t st);
void upconv_backward(const float* dout, int C, int H, int W, float* din, cudaStream_t st);
void mergecrop_backward(const float* dout, long long n, float* da, cudaStream_t st);
void softmax_backward(const double* prob, int C, int H, int W, int wp, const float* dout, float* din,
                      cudaStream_t st);
void sgd(float* w, float* mom, float* diff, long long n, float lr, float mu, float wd, cudaStream_t st);
void sgd(double* w, double* mom, double* diff, long long n, double lr, double mu, double wd, cudaStream_t st);
// softmax_loss (layers.hpp:269-307) over a [C][H][W] score blob (pitched): diff += gradient,
// *loss (device) = the reference's loss; terms = H*W f64 scratch; n_count = unmasked pixels.
void softmax_loss(const double* scores, int C, int H, int W, int wp, const int* labels,
                  const uint8_t* mask, long long n_count, float* diff, double* terms, double* loss,
                  cudaStream_t st);

// ---- gemm_i8.cu: exact integer GEMM on tcgen05 (kind::i8), C = A . B^T, K-major operands ----
void gemm_i8(const void* a, bool a_signed, const uint8_t* b, int M, int N, int K, int32_t* c,
             cudaStream_t st);

// ---- layers.cu ------------------------------------------------------------------------------
void f32_to_f64(const float* in, double* out, size_t n, cudaStream_t st);
void f64_to_f32(const double* in, float* out, size_t n, cudaStream_t st);

// maxpool_sk_forward (layers.hpp:102-132) over B x C planes; argmax nullable (per-image index).
// Row pitches (wp*, in doubles) default to compact rows when 0.
void f32_to_f64_pitched(const float* in, long long rows, int W, int wp, double* out,
                        cudaStream_t st);
void f64_pitched_to_f32(const double* in, long long rows, int W, int wp, float* out,
                        cudaStream_t st);
void maxpool(const double* in, int B, int C, int H, int W, int k, int d, int s, int OH, int OW,
             double* out, uint64_t* argmax, cudaStream_t st, int wpi = 0, int wpo = 0);
void relu(const double* in, double* out, size_t n, cudaStream_t st);
void upconv(const double* in, int B, int C, int H, int W, double* out, cudaStream_t st,
            int wpi = 0, int wpo = 0);
// mergecrop_forward (layers.hpp:196-212) for a batch: out[b] = a[b] ++ crop(b[b]).
void mergecrop(const double* a, int Ca, int Ha, int Wa, const double* b, int Cb, int Hb, int Wb,
               int B, double* out, cudaStream_t st, int wpa = 0, int wpb = 0, int wpo = 0);
// softmax_forward (layers.hpp:227-244); is_double selects S (the subtraction x-m in S).
void softmax(const double* in, int B, int C, int H, int W, double* out, bool is_double,
             cudaStream_t st, int wp = 0);
template <typename T>
void im2col(const T* in, int C, int H, int W, int k, int d, int s, int p, int OH, int OW, T* col,
            cudaStream_t st);
template <typename T>
void gemm(bool ta, bool tb, int m, int n, int k, T alpha, const T* a, const T* b, T beta, T* c,
          cudaStream_t st);
void mirror_pad_u8(const uint8_t* img, int H, int W, int v, uint8_t* out, cudaStream_t st);
void normalize_u8(const uint8_t* img, size_t n, float* out, cudaStream_t st);

// process() pieces (pipeline.hpp:654-694). Tiles are addressed by their row-major index in
// process()'s tiling: tile i sits at (min(y_base + (i / ntx) * w, H - w), min((i % ntx) * w,
// W - w)), the edge-snapping tile_offsets lambda (pipeline.hpp:662-672) started at y_base.
// Builds the inputs of tiles [t0, t0 + n_tiles) as n_tiles x f0 x (w+v) x (w+v) widened f32:
// mirror_pad + normalize_image + the f0-channel copy, straight from the raw u8 image.
// tiles_per_image > 0: a batch of same-size images stored back to back ([N][H][W]); global
// tile t belongs to image t / tiles_per_image.
void build_tiles(const uint8_t* img, int H, int W, int v, int w, int ntx, int t0, int n_tiles,
                 int f0, double* out, cudaStream_t st, int wp = 0, int y_base = 0,
                 int tiles_per_image = 0, int img_row0 = 0, long long img_plane = 0);
// Softmax head + per-pixel argmax + stitch of the tiles' scores (n_tiles x C x w x w) into the
// image planes: labels H x W (u8), probs C x H x W (f32); rows outside [y_lo, y_hi) skipped.
// A window of the planes (streamed process()): the buffers hold rows [out_row0, ...) of each
// plane, out_plane elements per plane (0: H * W). img_row0 / img_plane window the input image
// the same way for build_tiles.
void softmax_stitch(const double* scores, int n_tiles, int C, int w, int ntx, int t0, int H, int W,
                    int y_lo, int y_hi, uint8_t* labels, float* probs, cudaStream_t st, int wp = 0,
                    int y_base = 0, int tiles_per_image = 0, int out_row0 = 0, long long out_plane = 0);

// malis_softmax_loss (malis.hpp:311-346) for a batch of patches on device buffers (malis.cu):
// scores / sdiff [B][2][h][w] (sdiff accumulated), fg [B][h][w] u8, losses [B].
template <typename S>
void malis_softmax_loss_device(const S* scores, S* sdiff, const uint8_t* fg, int B, int h, int w, double* losses,
                               cudaStream_t st);

}  // namespace graft
