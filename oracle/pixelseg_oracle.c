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

/* ---- MALIS (malis.hpp): affinity graph, components, maximin gradient, composed loss ----- */

/* affinity_forward (malis.hpp:34-52): a = std::min(a, b), m = (b < a); unused last column /
 * row keep a = 1, m = 0. */
#define DEFINE_AFF_FWD(NAME, T)                                                              \
  void NAME(const T* img, int h, int w, T* ax, T* ay, uint8_t* mx, uint8_t* my) {            \
    for (int i = 0; i < h * w; ++i) { ax[i] = (T)1; ay[i] = (T)1; mx[i] = 0; my[i] = 0; }    \
    for (int y = 0; y < h; ++y)                                                              \
      for (int x = 0; x + 1 < w; ++x) {                                                      \
        const T a = img[y * w + x], b = img[y * w + x + 1];                                  \
        ax[y * w + x] = (b < a) ? b : a;                                                     \
        mx[y * w + x] = (b < a) ? 1 : 0;                                                     \
      }                                                                                      \
    for (int y = 0; y + 1 < h; ++y)                                                          \
      for (int x = 0; x < w; ++x) {                                                          \
        const T a = img[y * w + x], b = img[(y + 1) * w + x];                                \
        ay[y * w + x] = (b < a) ? b : a;                                                     \
        my[y * w + x] = (b < a) ? 1 : 0;                                                     \
      }                                                                                      \
  }
DEFINE_AFF_FWD(orc_affinity_forward_f32, float)
DEFINE_AFF_FWD(orc_affinity_forward_f64, double)

/* affinity_backward (malis.hpp:58-80): scatter in the reference's loop order. */
#define DEFINE_AFF_BWD(NAME, T)                                                              \
  void NAME(const T* dax, const T* day, const uint8_t* mx, const uint8_t* my, int h, int w,   \
            T* dpos, T* dneg) {                                                              \
    for (int i = 0; i < h * w; ++i) { dpos[i] = (T)0; dneg[i] = (T)0; }                      \
    for (int y = 0; y < h; ++y)                                                              \
      for (int x = 0; x + 1 < w; ++x) {                                                      \
        const int t = y * w + x + mx[y * w + x];                                             \
        dpos[t] += dax[y * w + x];                                                           \
        dneg[t] -= dax[y * w + x];                                                           \
      }                                                                                      \
    for (int y = 0; y + 1 < h; ++y)                                                          \
      for (int x = 0; x < w; ++x) {                                                          \
        const int t = (y + my[y * w + x]) * w + x;                                           \
        dpos[t] += day[y * w + x];                                                           \
        dneg[t] -= day[y * w + x];                                                           \
      }                                                                                      \
  }
DEFINE_AFF_BWD(orc_affinity_backward_f32, float)
DEFINE_AFF_BWD(orc_affinity_backward_f64, double)

/* connected_components (malis.hpp:84-111): breadth-first flood from each unlabelled nonzero
 * pixel in raster order, 4-neighbours in the order up, down, left, right. */
void orc_connected_components(const uint8_t* lab, int h, int w, int* comp) {
  const int n = h * w;
  int* queue = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  int next = 0;
  for (int i = 0; i < n; ++i) comp[i] = 0;
  for (int s = 0; s < n; ++s) {
    if (!lab[s] || comp[s]) continue;
    ++next;
    int qh = 0, qt = 0;
    queue[qt++] = s;
    comp[s] = next;
    while (qh < qt) {
      const int p = queue[qh++], y = p / w, x = p % w;
      const int ny[4] = {y - 1, y + 1, y, y}, nx[4] = {x, x, x - 1, x + 1};
      for (int k = 0; k < 4; ++k) {
        if (ny[k] < 0 || ny[k] >= h || nx[k] < 0 || nx[k] >= w) continue;
        const int q = ny[k] * w + nx[k];
        if (!lab[q] || comp[q]) continue;
        comp[q] = next;
        queue[qt++] = q;
      }
    }
  }
  free(queue);
}

/* PairTracker (malis.hpp:117-176): per set a sorted array of (component id, count). */
typedef struct {
  int* id;
  long long* n;
  int len, cap;
} orc_idmap;

static void idmap_merge(orc_idmap* a, orc_idmap* b, long long* pos, long long* bg) {
  /* pair counts of joining a and b (pos: same id > 0; bg: same id <= 0), then a += b */
  int* id = (int*)malloc(sizeof(int) * (size_t)(a->len + b->len));
  long long* n = (long long*)malloc(sizeof(long long) * (size_t)(a->len + b->len));
  int i = 0, j = 0, k = 0;
  *pos = 0;
  *bg = 0;
  while (i < a->len || j < b->len) {
    if (j >= b->len || (i < a->len && a->id[i] < b->id[j])) {
      id[k] = a->id[i]; n[k++] = a->n[i++];
    } else if (i >= a->len || b->id[j] < a->id[i]) {
      id[k] = b->id[j]; n[k++] = b->n[j++];
    } else {
      if (a->id[i] > 0) *pos += a->n[i] * b->n[j];
      else *bg += a->n[i] * b->n[j];
      id[k] = a->id[i]; n[k++] = a->n[i++] + b->n[j++];
    }
  }
  free(a->id); free(a->n); free(b->id); free(b->n);
  a->id = id; a->n = n; a->len = k; a->cap = k;
  b->id = NULL; b->n = NULL; b->len = 0; b->cap = 0;
}

typedef struct {
  const void* val; /* edge values (float or double) */
  int dbl;
} orc_edge_cmp_ctx;
static __thread orc_edge_cmp_ctx g_cmp;
static int edge_cmp(const void* pa, const void* pb) {
  const int i = *(const int*)pa, j = *(const int*)pb;
  const double vi = g_cmp.dbl ? ((const double*)g_cmp.val)[i] : (double)((const float*)g_cmp.val)[i];
  const double vj = g_cmp.dbl ? ((const double*)g_cmp.val)[j] : (double)((const float*)g_cmp.val)[j];
  if (vi != vj) return vi > vj ? -1 : 1;
  return i < j ? -1 : (i > j ? 1 : 0);
}

static int uf_root(int* parent, int v) {
  while (parent[v] != v) {
    parent[v] = parent[parent[v]];
    v = parent[v];
  }
  return v;
}

/* malis_gradient (malis.hpp:197-298). Edge ids: horizontal edges in raster order, then
 * vertical. Outputs zeroed first; totals[2], losses[3] = {pos, neg, total}. */
#define DEFINE_MALIS(NAME, T, DBL)                                                           \
  void NAME(const T* pax, const T* pay, const T* tax, const T* tay, const int* comp, int h,   \
            int w, T* dax, T* day, long long* posx, long long* posy, long long* negx,        \
            long long* negy, long long* totals, double* losses) {                            \
    const int n = h * w, nx = h * (w > 0 ? w - 1 : 0), ne = nx + (h > 0 ? h - 1 : 0) * w;     \
    for (int i = 0; i < n; ++i) {                                                            \
      dax[i] = (T)0; day[i] = (T)0; posx[i] = posy[i] = negx[i] = negy[i] = 0;               \
    }                                                                                        \
    int *ea = (int*)malloc(sizeof(int) * (ne + 1)), *eb = (int*)malloc(sizeof(int) * (ne + 1)); \
    int* epos = (int*)malloc(sizeof(int) * (ne + 1));                                        \
    for (int y = 0, e = 0; y < h; ++y)                                                       \
      for (int x = 0; x + 1 < w; ++x, ++e) { ea[e] = y * w + x; eb[e] = ea[e] + 1; epos[e] = ea[e]; } \
    for (int y = 0, e = nx; y + 1 < h; ++y)                                                  \
      for (int x = 0; x < w; ++x, ++e) { ea[e] = y * w + x; eb[e] = ea[e] + w; epos[e] = ea[e]; } \
    T* val = (T*)malloc(sizeof(T) * (ne + 1));                                               \
    int* order = (int*)malloc(sizeof(int) * (ne + 1));                                       \
    long long* cnt = (long long*)malloc(sizeof(long long) * (ne + 1));                       \
    double* graw = (double*)malloc(sizeof(double) * (ne + 1));                               \
    int *parent = (int*)malloc(sizeof(int) * (n + 1)), *rnk = (int*)malloc(sizeof(int) * (n + 1)); \
    long long* size = (long long*)malloc(sizeof(long long) * (n + 1));                       \
    orc_idmap* maps = (orc_idmap*)calloc((size_t)n + 1, sizeof(orc_idmap));                  \
    double loss[2] = {0, 0};                                                                 \
    for (int pass = 0; pass < 2; ++pass) {                                                   \
      const int positive = pass == 0;                                                        \
      for (int e = 0; e < ne; ++e) {                                                         \
        const T p = e < nx ? pax[epos[e]] : pay[epos[e]];                                    \
        const T t = e < nx ? tax[epos[e]] : tay[epos[e]];                                    \
        val[e] = positive ? ((t < p) ? t : p) : ((p < t) ? t : p);                            \
        order[e] = e;                                                                        \
        cnt[e] = 0;                                                                          \
        graw[e] = 0.0;                                                                       \
      }                                                                                      \
      g_cmp.val = val;                                                                       \
      g_cmp.dbl = DBL;                                                                       \
      qsort(order, (size_t)ne, sizeof(int), edge_cmp);                                       \
      for (int i = 0; i < n; ++i) {                                                          \
        parent[i] = i; rnk[i] = 0; size[i] = 1;                                              \
        free(maps[i].id); free(maps[i].n);                                                   \
        maps[i].id = (int*)malloc(sizeof(int)); maps[i].n = (long long*)malloc(sizeof(long long)); \
        maps[i].id[0] = comp[i]; maps[i].n[0] = 1; maps[i].len = maps[i].cap = 1;            \
      }                                                                                      \
      long long total = 0;                                                                   \
      double loss_raw = 0.0;                                                                 \
      for (int r = 0; r < ne; ++r) {                                                         \
        const int e = order[r];                                                              \
        int ra = uf_root(parent, ea[e]), rb = uf_root(parent, eb[e]);                        \
        if (ra == rb) continue;                                                              \
        const long long sa = size[ra], sb = size[rb];                                        \
        if (rnk[ra] < rnk[rb]) { const int t = ra; ra = rb; rb = t; }                        \
        long long pos, bg;                                                                   \
        idmap_merge(&maps[ra], &maps[rb], &pos, &bg);                                        \
        parent[rb] = ra;                                                                     \
        if (rnk[ra] == rnk[rb]) ++rnk[ra];                                                   \
        size[ra] = sa + sb;                                                                  \
        const long long neg = sa * sb - pos - bg;                                            \
        const long long c = positive ? pos : neg;                                            \
        if (c == 0) continue;                                                                \
        cnt[e] = c;                                                                          \
        total += c;                                                                          \
        const double a = (double)val[e];                                                     \
        if (positive) {                                                                      \
          loss_raw += (double)c * (1.0 - a) * (1.0 - a);                                     \
          graw[e] = (double)c * (-2.0) * (1.0 - a);                                          \
        } else {                                                                             \
          loss_raw += (double)c * a * a;                                                     \
          graw[e] = (double)c * 2.0 * a;                                                     \
        }                                                                                    \
      }                                                                                      \
      const double norm = total > 0 ? 1.0 / (double)total : 0.0;                             \
      for (int e = 0; e < ne; ++e) {                                                         \
        if (cnt[e] == 0) continue;                                                           \
        const int hz = e < nx;                                                               \
        long long* counts = hz ? (positive ? posx : negx) : (positive ? posy : negy);        \
        counts[epos[e]] = cnt[e];                                                            \
        const T p = hz ? pax[epos[e]] : pay[epos[e]], t = hz ? tax[epos[e]] : tay[epos[e]];   \
        if (positive ? (p <= t) : (p >= t)) {                                                \
          T* da = hz ? dax : day;                                                            \
          da[epos[e]] += (T)(graw[e] * norm);                                                \
        }                                                                                    \
      }                                                                                      \
      totals[pass] = total;                                                                  \
      loss[pass] = loss_raw * norm;                                                          \
    }                                                                                        \
    losses[0] = loss[0];                                                                     \
    losses[1] = loss[1];                                                                     \
    losses[2] = loss[0] + loss[1];                                                           \
    for (int i = 0; i < n; ++i) { free(maps[i].id); free(maps[i].n); }                       \
    free(maps); free(ea); free(eb); free(epos); free(val); free(order); free(cnt); free(graw); \
    free(parent); free(rnk); free(size);                                                     \
  }
DEFINE_MALIS(orc_malis_gradient_f32, float, 0)
DEFINE_MALIS(orc_malis_gradient_f64, double, 1)

/* malis_softmax_loss (malis.hpp:311-346); diff [2][h][w] accumulated. */
#define DEFINE_MALIS_LOSS(NAME, T, SOFTMAX, AFF, GRAD, BWD)                                   \
  int NAME(const T* scores, int C, int h, int w, const uint8_t* fg, T* diff, double* loss) {  \
    if (C != 2) return fail(ORC_ESIZE, "malis loss: needs exactly 2 score channels, got %d", C); \
    const size_t n = (size_t)h * w, nn = n ? n : 1;                                          \
    T* probs = (T*)malloc(sizeof(T) * 2 * nn);                                               \
    T* ft = (T*)malloc(sizeof(T) * nn);                                                      \
    T *pax = (T*)malloc(sizeof(T) * nn), *pay = (T*)malloc(sizeof(T) * nn);                  \
    T *tax = (T*)malloc(sizeof(T) * nn), *tay = (T*)malloc(sizeof(T) * nn);                  \
    T *dax = (T*)malloc(sizeof(T) * nn), *day = (T*)malloc(sizeof(T) * nn);                  \
    T *dp = (T*)malloc(sizeof(T) * nn), *dn = (T*)malloc(sizeof(T) * nn);                    \
    uint8_t *mx = (uint8_t*)malloc(nn), *my = (uint8_t*)malloc(nn), *tmx = (uint8_t*)malloc(nn), \
            *tmy = (uint8_t*)malloc(nn);                                                     \
    int* comp = (int*)malloc(sizeof(int) * nn);                                              \
    long long* cnts = (long long*)malloc(sizeof(long long) * 4 * nn);                        \
    long long totals[2];                                                                     \
    double losses[3];                                                                        \
    SOFTMAX(scores, 2, h, w, probs);                                                         \
    for (size_t i = 0; i < n; ++i) ft[i] = fg[i] ? (T)1 : (T)0;                              \
    AFF(probs + n, h, w, pax, pay, mx, my);                                                  \
    AFF(ft, h, w, tax, tay, tmx, tmy);                                                       \
    orc_connected_components(fg, h, w, comp);                                                \
    GRAD(pax, pay, tax, tay, comp, h, w, dax, day, cnts, cnts + nn, cnts + 2 * nn,           \
         cnts + 3 * nn, totals, losses);                                                     \
    BWD(dax, day, mx, my, h, w, dp, dn);                                                     \
    for (size_t px = 0; px < n; ++px) {                                                      \
      const T g1 = dp[px] * (T)0.5, g0 = dn[px] * (T)0.5;                                    \
      double mix = 0.0;                                                                      \
      mix += (double)g0 * (double)probs[px];                                                 \
      mix += (double)g1 * (double)probs[n + px];                                             \
      diff[px] += (T)((double)probs[px] * ((double)g0 - mix));                               \
      diff[n + px] += (T)((double)probs[n + px] * ((double)g1 - mix));                       \
    }                                                                                        \
    *loss = losses[2];                                                                       \
    free(probs); free(ft); free(pax); free(pay); free(tax); free(tay); free(dax); free(day);  \
    free(dp); free(dn); free(mx); free(my); free(tmx); free(tmy); free(comp); free(cnts);    \
    return ORC_OK;                                                                           \
  }
DEFINE_MALIS_LOSS(orc_malis_softmax_loss_f32, float, orc_softmax_f32, orc_affinity_forward_f32,
                  orc_malis_gradient_f32, orc_affinity_backward_f32)
DEFINE_MALIS_LOSS(orc_malis_softmax_loss_f64, double, orc_softmax_f64, orc_affinity_forward_f64,
                  orc_malis_gradient_f64, orc_affinity_backward_f64)
