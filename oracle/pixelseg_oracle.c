/*
 * pixelseg_oracle.c -- plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pixelseg_oracle.h): used by tests/, smoke() and the
 * cpu_baseline leg of bench.py as the checker. Every function cites the reference
 * file:line (under /root/reference/proj/include/pixelseg/ unless stated) it restates.
 *
 * Build: oracle/Makefile, `-O2 -ffp-contract=off` so double arithmetic is the plain
 * mul-then-add sequence the reference's x86-64 build (no -march, no FMA) performs.
 */
#include "pixelseg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ------------------------------------------------------------------------------------------
 * Rng (rng.hpp:12-54): std::mt19937_64 (the standard's parameters), uniform = (u64>>11)*2^-53,
 * uniform(lo,hi) = lo + (hi-lo)*u, uniform_index = u64 % n, gaussian = Box-Muller with a cached
 * spare (sin branch) returning the cos branch first.
 * ---------------------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

size_t orc_rng_state_size(void) { return sizeof(orc_rng); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
  r->spare = 0.0;
  r->have_spare = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      const uint64_t y = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    }
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_uniform01(r);
}

uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

double orc_rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  do {
    u1 = orc_rng_uniform01(r);
  } while (u1 <= 0.0);
  const double u2 = orc_rng_uniform01(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

double orc_rng_gaussian_ms(orc_rng* r, double mean, double sigma) {
  return mean + sigma * orc_rng_gaussian(r);
}

void orc_rng_fill_uniform_f32(orc_rng* r, float* dst, size_t n, double lo, double hi) {
  for (size_t i = 0; i < n; ++i) dst[i] = (float)orc_rng_uniform(r, lo, hi);
}
void orc_rng_fill_uniform_f64(orc_rng* r, double* dst, size_t n, double lo, double hi) {
  for (size_t i = 0; i < n; ++i) dst[i] = orc_rng_uniform(r, lo, hi);
}
void orc_rng_fill_gaussian_f32(orc_rng* r, float* dst, size_t n, double mean, double sigma) {
  for (size_t i = 0; i < n; ++i) dst[i] = (float)orc_rng_gaussian_ms(r, mean, sigma);
}
void orc_rng_fill_gaussian_f64(orc_rng* r, double* dst, size_t n, double mean, double sigma) {
  for (size_t i = 0; i < n; ++i) dst[i] = orc_rng_gaussian_ms(r, mean, sigma);
}
void orc_rng_fill_index_u8(orc_rng* r, uint8_t* dst, size_t n, uint64_t m) {
  for (size_t i = 0; i < n; ++i) dst[i] = (uint8_t)orc_rng_uniform_index(r, m);
}

/* ------------------------------------------------------------------------------------------
 * ConvGeometry::out_extent (tensor.hpp:26-42): span = (k-1)d+1; out = (in+2p-span)/s + 1, the
 * division exact, else SizeError. Messages are the reference's verbatim.
 * ---------------------------------------------------------------------------------------- */
int orc_out_extent(int in, int k, int d, int s, int p, const char* what, int* out) {
  const int span = (k - 1) * d + 1;
  if (k < 1 || d < 1 || s < 1 || p < 0) {
    return fail(ORC_ESIZE, "%s: require k,d,s >= 1 and p >= 0", what);
  }
  const int padded = in + 2 * p;
  if (span > padded) {
    return fail(ORC_ESIZE, "%s: kernel span %d exceeds padded input %d", what, span, padded);
  }
  const int num = padded - span;
  if (num % s != 0) {
    return fail(ORC_ESIZE, "%s: input %d with span %d not divisible by stride %d", what, in, span,
                s);
  }
  *out = num / s + 1;
  return ORC_OK;
}

static int geometry(int H, int W, int k, int d, int s, int p, int* oh, int* ow) {
  int rc = orc_out_extent(H, k, d, s, p, "height", oh);
  if (rc) return rc;
  return orc_out_extent(W, k, d, s, p, "width", ow);
}

/* ------------------------------------------------------------------------------------------
 * im2col_sk (tensor.hpp:80-110): row r = (c*k+ky)*k+kx, column n = oy*ow+ox holds
 * in[c, oy*s+ky*d-p, ox*s+kx*d-p] or 0 outside.
 * ---------------------------------------------------------------------------------------- */
#define DEFINE_IM2COL(NAME, T)                                                               \
  int NAME(const T* in, int C, int H, int W, int k, int d, int s, int p, T* col) {           \
    int oh, ow;                                                                              \
    int rc = geometry(H, W, k, d, s, p, &oh, &ow);                                           \
    if (rc) return rc;                                                                       \
    size_t r = 0;                                                                            \
    for (int c = 0; c < C; ++c)                                                              \
      for (int ky = 0; ky < k; ++ky)                                                         \
        for (int kx = 0; kx < k; ++kx, ++r) {                                                \
          T* dst = col + r * (size_t)oh * ow;                                                \
          for (int oy = 0; oy < oh; ++oy) {                                                  \
            const int iy = oy * s + ky * d - p;                                              \
            for (int ox = 0; ox < ow; ++ox) {                                                \
              const int ix = ox * s + kx * d - p;                                            \
              *dst++ = (iy >= 0 && iy < H && ix >= 0 && ix < W)                              \
                           ? in[((size_t)c * H + iy) * W + ix]                               \
                           : (T)0;                                                           \
            }                                                                                \
          }                                                                                  \
        }                                                                                    \
    return ORC_OK;                                                                           \
  }
DEFINE_IM2COL(orc_im2col_f32, float)
DEFINE_IM2COL(orc_im2col_f64, double)

/* ------------------------------------------------------------------------------------------
 * gemm (tensor.hpp:151-169): acc += double(a)*double(b) for kk ascending from 0.0;
 * r = double(alpha)*acc; if beta != 0: r += double(beta)*double(c); c = S(r).
 * ---------------------------------------------------------------------------------------- */
#define DEFINE_GEMM(NAME, T)                                                                 \
  void NAME(int ta, int tb, int m, int n, int k, T alpha, const T* a, const T* b, T beta,    \
            T* c) {                                                                          \
    const size_t lda = ta ? (size_t)m : (size_t)k;                                           \
    const size_t ldb = tb ? (size_t)k : (size_t)n;                                           \
    for (int i = 0; i < m; ++i)                                                              \
      for (int j = 0; j < n; ++j) {                                                          \
        double acc = 0.0;                                                                    \
        for (int kk = 0; kk < k; ++kk) {                                                     \
          const T av = ta ? a[(size_t)kk * lda + i] : a[(size_t)i * lda + kk];               \
          const T bv = tb ? b[(size_t)j * ldb + kk] : b[(size_t)kk * ldb + j];               \
          acc += (double)av * (double)bv;                                                    \
        }                                                                                    \
        double r = (double)alpha * acc;                                                      \
        if (beta != (T)0) r += (double)beta * (double)c[(size_t)i * n + j];                  \
        c[(size_t)i * n + j] = (T)r;                                                         \
      }                                                                                      \
  }
DEFINE_GEMM(orc_gemm_f32, float)
DEFINE_GEMM(orc_gemm_f64, double)

/* ------------------------------------------------------------------------------------------
 * conv_sk_forward (layers.hpp:43-64) restated as the direct loop of the reference's test
 * oracle ref_conv (tests/oracles.hpp:51-82): per output, taps in (c,ky,kx) order into a
 * double, out = S(acc) then += bias in S. Out-of-range taps contribute exactly nothing in
 * the reference too (acc + (+-0) == acc, acc never -0 from a +0 start).
 * ---------------------------------------------------------------------------------------- */
#define DEFINE_CONV_RANGE(NAME, T)                                                           \
  static void NAME(const T* in, int C, int H, int W, const T* w, const T* b, int f0, int f1, \
                   int k, int d, int s, int p, int oh, int ow, T* out) {                     \
    const int taps = C * k * k;                                                              \
    for (int fo = f0; fo < f1; ++fo) {                                                       \
      const T* wrow = w + (size_t)fo * taps;                                                 \
      for (int oy = 0; oy < oh; ++oy)                                                        \
        for (int ox = 0; ox < ow; ++ox) {                                                    \
          double acc = 0.0;                                                                  \
          int r = 0;                                                                         \
          for (int c = 0; c < C; ++c)                                                        \
            for (int ky = 0; ky < k; ++ky)                                                   \
              for (int kx = 0; kx < k; ++kx, ++r) {                                          \
                const int iy = oy * s + ky * d - p;                                          \
                const int ix = ox * s + kx * d - p;                                          \
                if (iy >= 0 && iy < H && ix >= 0 && ix < W)                                  \
                  acc += (double)wrow[r] * (double)in[((size_t)c * H + iy) * W + ix];        \
              }                                                                              \
          T v = (T)acc;                                                                      \
          v += b[fo];                                                                        \
          out[((size_t)fo * oh + oy) * ow + ox] = v;                                         \
        }                                                                                    \
    }                                                                                        \
  }
DEFINE_CONV_RANGE(conv_range_f32, float)
DEFINE_CONV_RANGE(conv_range_f64, double)

int orc_conv_f32(const float* in, int C, int H, int W, const float* w, const float* b, int f_out,
                 int k, int d, int s, int p, float* out) {
  int oh, ow;
  int rc = geometry(H, W, k, d, s, p, &oh, &ow);
  if (rc) return rc;
  conv_range_f32(in, C, H, W, w, b, 0, f_out, k, d, s, p, oh, ow, out);
  return ORC_OK;
}

int orc_conv_f64(const double* in, int C, int H, int W, const double* w, const double* b,
                 int f_out, int k, int d, int s, int p, double* out) {
  int oh, ow;
  int rc = geometry(H, W, k, d, s, p, &oh, &ow);
  if (rc) return rc;
  conv_range_f64(in, C, H, W, w, b, 0, f_out, k, d, s, p, oh, ow, out);
  return ORC_OK;
}

typedef struct {
  const float *in, *w, *b;
  float* out;
  int C, H, W, k, d, s, p, oh, ow, f0, f1;
} conv_job;

static void* conv_worker(void* arg) {
  conv_job* j = (conv_job*)arg;
  conv_range_f32(j->in, j->C, j->H, j->W, j->w, j->b, j->f0, j->f1, j->k, j->d, j->s, j->p, j->oh,
                 j->ow, j->out);
  return NULL;
}

int orc_conv_f32_mt(const float* in, int C, int H, int W, const float* w, const float* b, int f_out,
                    int k, int d, int s, int p, float* out, int nthreads) {
  int oh, ow;
  int rc = geometry(H, W, k, d, s, p, &oh, &ow);
  if (rc) return rc;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > f_out) nthreads = f_out;
  pthread_t th[256];
  conv_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    conv_job j = {in, w, b, out, C, H, W, k, d, s, p, oh, ow, (int)((long)f_out * t / nthreads),
                  (int)((long)f_out * (t + 1) / nthreads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, conv_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------
 * maxpool_sk_forward (layers.hpp:102-132): taps at (oy*s+ky*d, ox*s+kx*d) -- no padding term;
 * first tap seeds, strict '>' afterwards, so ties keep the smallest input linear index.
 * ---------------------------------------------------------------------------------------- */
#define DEFINE_POOL(NAME, T)                                                                 \
  int NAME(const T* in, int C, int H, int W, int k, int d, int s, T* out, uint64_t* argmax) { \
    int oh, ow;                                                                              \
    int rc = geometry(H, W, k, d, s, 0, &oh, &ow);                                           \
    if (rc) return rc;                                                                       \
    size_t o = 0;                                                                            \
    for (int c = 0; c < C; ++c)                                                              \
      for (int oy = 0; oy < oh; ++oy)                                                        \
        for (int ox = 0; ox < ow; ++ox, ++o) {                                               \
          T best = (T)0;                                                                     \
          size_t best_idx = 0;                                                               \
          int first = 1;                                                                     \
          for (int ky = 0; ky < k; ++ky) {                                                   \
            const int iy = oy * s + ky * d;                                                  \
            for (int kx = 0; kx < k; ++kx) {                                                 \
              const int ix = ox * s + kx * d;                                                \
              const size_t idx = ((size_t)c * H + iy) * W + ix;                              \
              const T v = in[idx];                                                           \
              if (first || v > best) {                                                       \
                best = v;                                                                    \
                best_idx = idx;                                                              \
                first = 0;                                                                   \
              }                                                                              \
            }                                                                                \
          }                                                                                  \
          out[o] = best;                                                                     \
          if (argmax) argmax[o] = best_idx;                                                  \
        }                                                                                    \
    return ORC_OK;                                                                           \
  }
DEFINE_POOL(orc_maxpool_f32, float)
DEFINE_POOL(orc_maxpool_f64, double)

/* relu_forward (layers.hpp:143-147): in > 0 ? in : 0 (so -0 and NaN map to +0). */
void orc_relu_f32(const float* in, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = in[i] > 0.0f ? in[i] : 0.0f;
}
void orc_relu_f64(const double* in, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = in[i] > 0.0 ? in[i] : 0.0;
}

/* upconv_forward (layers.hpp:162-176): nearest-neighbour 2x replication. */
#define DEFINE_UPCONV(NAME, T)                                                               \
  void NAME(const T* in, int C, int H, int W, T* out) {                                      \
    const int OW = 2 * W;                                                                    \
    for (int c = 0; c < C; ++c)                                                              \
      for (int y = 0; y < H; ++y)                                                            \
        for (int x = 0; x < W; ++x) {                                                        \
          const T v = in[((size_t)c * H + y) * W + x];                                       \
          T* o = out + ((size_t)c * 2 * H + 2 * y) * OW + 2 * x;                             \
          o[0] = v;                                                                          \
          o[1] = v;                                                                          \
          o[OW] = v;                                                                         \
          o[OW + 1] = v;                                                                     \
        }                                                                                    \
  }
DEFINE_UPCONV(orc_upconv_f32, float)
DEFINE_UPCONV(orc_upconv_f64, double)

/* mergecrop_forward (layers.hpp:196-212): A's channels, then B cropped at floor((B-A)/2). */
#define DEFINE_MERGECROP(NAME, T)                                                            \
  int NAME(const T* a, int Ca, int Ha, int Wa, const T* b, int Cb, int Hb, int Wb, T* out) { \
    if (Hb < Ha || Wb < Wa) {                                                                \
      return fail(ORC_ESIZE, "mergecrop: second input %dx%d smaller than first %dx%d", Hb,  \
                  Wb, Ha, Wa);                                                               \
    }                                                                                        \
    const int oy = (Hb - Ha) / 2, ox = (Wb - Wa) / 2;                                        \
    const size_t plane = (size_t)Ha * Wa;                                                    \
    memcpy(out, a, sizeof(T) * plane * Ca);                                                  \
    for (int c = 0; c < Cb; ++c)                                                             \
      for (int y = 0; y < Ha; ++y)                                                           \
        for (int x = 0; x < Wa; ++x)                                                         \
          out[(size_t)(Ca + c) * plane + (size_t)y * Wa + x] =                               \
              b[((size_t)c * Hb + y + oy) * Wb + x + ox];                                    \
    return ORC_OK;                                                                           \
  }
DEFINE_MERGECROP(orc_mergecrop_f32, float)
DEFINE_MERGECROP(orc_mergecrop_f64, double)

/* softmax_forward (layers.hpp:227-244): m = std::max over channels in S; e = exp(double(x-m))
 * with (x-m) rounded in S; out = S(e); sum += e (double); out = S(double(out)/sum). */
#define DEFINE_SOFTMAX(NAME, T)                                                              \
  void NAME(const T* in, int C, int H, int W, T* out) {                                      \
    const size_t plane = (size_t)H * W;                                                      \
    for (size_t px = 0; px < plane; ++px) {                                                  \
      T m = in[px];                                                                          \
      for (int c = 1; c < C; ++c) {                                                          \
        const T x = in[(size_t)c * plane + px];                                              \
        m = (m < x) ? x : m; /* std::max(m, x) */                                            \
      }                                                                                      \
      double sum = 0.0;                                                                      \
      for (int c = 0; c < C; ++c) {                                                          \
        const T diff = in[(size_t)c * plane + px] - m;                                       \
        const double e = exp((double)diff);                                                  \
        out[(size_t)c * plane + px] = (T)e;                                                  \
        sum += e;                                                                            \
      }                                                                                      \
      for (int c = 0; c < C; ++c)                                                            \
        out[(size_t)c * plane + px] = (T)((double)out[(size_t)c * plane + px] / sum);        \
    }                                                                                        \
  }
DEFINE_SOFTMAX(orc_softmax_f32, float)
DEFINE_SOFTMAX(orc_softmax_f64, double)

/* mirror_pad (pipeline.hpp:36-58): ceil(v/2) before, floor(v/2) after, reflection without
 * repeating the border pixel. */
int orc_mirror_pad_u8(const uint8_t* img, int H, int W, int v, uint8_t* out) {
  if (v < 0) return fail(ORC_ESIZE, "mirror_pad: negative padding");
  if (v == 0) {
    memcpy(out, img, (size_t)H * W);
    return ORC_OK;
  }
  const int before = (v + 1) / 2;
  if (before > H - 1 || before > W - 1) {
    return fail(ORC_ESIZE, "mirror_pad: padding %d needs an image larger than %d pixels", before,
                before + 1);
  }
  const int OH = H + v, OW = W + v;
  for (int y = 0; y < OH; ++y) {
    int sy = y - before;
    if (sy < 0) sy = -sy;
    if (sy >= H) sy = 2 * H - 2 - sy;
    for (int x = 0; x < OW; ++x) {
      int sx = x - before;
      if (sx < 0) sx = -sx;
      if (sx >= W) sx = 2 * W - 2 - sx;
      out[(size_t)y * OW + x] = img[(size_t)sy * W + sx];
    }
  }
  return ORC_OK;
}

/* normalize_image (pipeline.hpp:86-93): S(double(x)/127.5 - 1.0). */
void orc_normalize_f32(const uint8_t* img, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)((double)img[i] / 127.5 - 1.0);
}
void orc_normalize_f64(const uint8_t* img, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (double)img[i] / 127.5 - 1.0;
}

/* tile_offsets lambda (pipeline.hpp:662-672): steps of w, the last tile snapped to extent-w. */
int orc_tile_offsets(int extent, int w, int* offs, int cap) {
  int n = 0;
  for (int o = 0;; o += w) {
    if (o + w >= extent) {
      if (n < cap) offs[n] = extent - w;
      ++n;
      break;
    }
    if (n < cap) offs[n] = o;
    ++n;
  }
  return n;
}

/* argmax + stitch (pipeline.hpp:685-694): best = first class with strictly larger prob. */
void orc_stitch_f32(const float* tp, int C, int w, int oy, int ox, int H, int W, uint8_t* labels,
                    float* probs) {
  const size_t tplane = (size_t)w * w, plane = (size_t)H * W;
  for (int y = 0; y < w; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t t = (size_t)y * w + x;
      int best = 0;
      for (int c = 1; c < C; ++c)
        if (tp[(size_t)c * tplane + t] > tp[(size_t)best * tplane + t]) best = c;
      const size_t o = (size_t)(oy + y) * W + (ox + x);
      labels[o] = (uint8_t)best;
      for (int c = 0; c < C; ++c) probs[(size_t)c * plane + o] = tp[(size_t)c * tplane + t];
    }
}
