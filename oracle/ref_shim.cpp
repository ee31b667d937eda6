// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference headers
// (/root/reference/proj/include/pixelseg/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libpixelseg_ref.so. TEST INFRASTRUCTURE ONLY: it lets tests/golden/make_golden.py
// produce golden vectors from the reference itself, pins the C restatement
// (oracle/pixelseg_oracle.c) against the reference, and is the "reference" CPU baseline of
// bench.py --impl reference. No reference source is copied here; the headers are included
// from where they lie, with the reference's own build flags (-std=c++20 -O3 -DNDEBUG,
// proj/CMakeLists.txt:3-10).
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pixelseg/convert.hpp"
#include "pixelseg/image_io.hpp"
#include "pixelseg/layers.hpp"
#include "pixelseg/malis.hpp"
#include "pixelseg/netgraph.hpp"
#include "pixelseg/netspec.hpp"
#include "pixelseg/pipeline.hpp"
#include "pixelseg/tensor.hpp"
#include "pixelseg/weights_io.hpp"

using namespace pixelseg;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const SizeError& e) {
    g_err = e.what();
    return 6;
  } catch (const SpecError& e) {
    g_err = e.what();
    return 2;
  } catch (const IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

template <typename S>
Blob<S> make_blob(const S* p, int c, int h, int w) {
  Blob<S> b(c, h, w);
  std::memcpy(b.data.data(), p, b.size() * sizeof(S));
  return b;
}

struct RefNet {
  NetSpec spec;
  NetStates<float> states;
  std::unique_ptr<NetRunner<float>> runner;
  Blob<float> last;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_im2col_f32(const float* in, int C, int H, int W, int k, int d, int s, int p, float* col) {
  return guard([&] {
    const Blob<float> b = make_blob(in, C, H, W);
    const ConvGeometry g = ConvGeometry::from_input(k, d, s, p, H, W);
    ColumnBuffer<float> cb;
    im2col_sk(b, g, cb);
    std::memcpy(col, cb.data.data(), sizeof(float) * cb.rows * cb.cols);
  });
}

void ref_gemm_f32(int ta, int tb, int m, int n, int k, float alpha, const float* a, const float* b,
                  float beta, float* c) {
  gemm<float>(ta != 0, tb != 0, m, n, k, alpha, a, b, beta, c);
}

void ref_gemm_f64(int ta, int tb, int m, int n, int k, double alpha, const double* a,
                  const double* b, double beta, double* c) {
  gemm<double>(ta != 0, tb != 0, m, n, k, alpha, a, b, beta, c);
}

#define REF_CONV(NAME, S)                                                                       \
  int NAME(const S* in, int C, int H, int W, const S* w, const S* bias, int f_out, int k, int d, \
           int s, int p, S* out) {                                                              \
    return guard([&] {                                                                          \
      const Blob<S> b = make_blob(in, C, H, W);                                                 \
      LayerState<S> st;                                                                         \
      st.init_conv(f_out, C * k * k);                                                           \
      std::memcpy(st.weights.data(), w, sizeof(S) * st.weights.size());                         \
      std::memcpy(st.bias.data(), bias, sizeof(S) * st.bias.size());                            \
      const ConvGeometry g = ConvGeometry::from_input(k, d, s, p, H, W);                        \
      ColumnBuffer<S> cb;                                                                       \
      Blob<S> o;                                                                                \
      conv_sk_forward(b, st, f_out, g, cb, o);                                                  \
      std::memcpy(out, o.data.data(), sizeof(S) * o.size());                                    \
    });                                                                                         \
  }
REF_CONV(ref_conv_f32, float)
REF_CONV(ref_conv_f64, double)

int ref_maxpool_f32(const float* in, int C, int H, int W, int k, int d, int s, float* out,
                    uint64_t* argmax) {
  return guard([&] {
    const Blob<float> b = make_blob(in, C, H, W);
    const ConvGeometry g = ConvGeometry::from_input(k, d, s, 0, H, W);
    LayerState<float> st;
    Blob<float> o;
    maxpool_sk_forward(b, st, g, o);
    std::memcpy(out, o.data.data(), sizeof(float) * o.size());
    if (argmax)
      for (std::size_t i = 0; i < st.argmax.size(); ++i) argmax[i] = st.argmax[i];
  });
}

void ref_relu_f32(const float* in, int C, int H, int W, float* out) {
  const Blob<float> b = make_blob(in, C, H, W);
  Blob<float> o;
  relu_forward(b, o);
  std::memcpy(out, o.data.data(), sizeof(float) * o.size());
}

void ref_upconv_f32(const float* in, int C, int H, int W, float* out) {
  const Blob<float> b = make_blob(in, C, H, W);
  Blob<float> o;
  upconv_forward(b, o);
  std::memcpy(out, o.data.data(), sizeof(float) * o.size());
}

int ref_mergecrop_f32(const float* a, int Ca, int Ha, int Wa, const float* b, int Cb, int Hb,
                      int Wb, float* out) {
  return guard([&] {
    const Blob<float> A = make_blob(a, Ca, Ha, Wa);
    const Blob<float> B = make_blob(b, Cb, Hb, Wb);
    Blob<float> o;
    mergecrop_forward(A, B, o);
    std::memcpy(out, o.data.data(), sizeof(float) * o.size());
  });
}

void ref_softmax_f32(const float* in, int C, int H, int W, float* out) {
  const Blob<float> b = make_blob(in, C, H, W);
  Blob<float> o;
  softmax_forward(b, o);
  std::memcpy(out, o.data.data(), sizeof(float) * o.size());
}

int ref_mirror_pad_u8(const uint8_t* img, int H, int W, int v, uint8_t* out) {
  return guard([&] {
    Plane<std::uint8_t> p(H, W);
    std::memcpy(p.pix.data(), img, p.size());
    const Plane<std::uint8_t> o = mirror_pad(p, v);
    std::memcpy(out, o.pix.data(), o.size());
  });
}

void ref_normalize_f32(const uint8_t* img, int n, float* out) {
  Plane<std::uint8_t> p(1, n);
  std::memcpy(p.pix.data(), img, n);
  const Plane<float> o = normalize_image<float>(p);
  std::memcpy(out, o.pix.data(), sizeof(float) * n);
}

// ---- net-level entry points ----
void* ref_net_create(const char* text) {
  RefNet* n = nullptr;
  const int rc = guard([&] {
    n = new RefNet;
    n->spec = parse_netspec_or_throw(text);
  });
  if (rc) {
    delete n;
    return nullptr;
  }
  return n;
}

void ref_net_destroy(void* h) { delete static_cast<RefNet*>(h); }

// Returns the corrected spec text of a sliding-window net (convert.hpp:175-195) into buf.
int ref_correct_sw(const char* text, char* buf, int cap) {
  return guard([&] {
    const NetSpec s = correct_sw(parse_netspec_or_throw(text));
    const std::string out = write_netspec(s);
    if (static_cast<int>(out.size()) + 1 > cap) throw SpecError("buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

int ref_net_init_weights(void* h, uint64_t seed) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    n->states = init_weights<float>(n->spec, seed);
    n->runner.reset();
  });
}

int ref_net_num_layers(void* h) { return static_cast<int>(static_cast<RefNet*>(h)->spec.layers.size()); }

// weights/bias sizes of a layer (0 for parameterless layers)
void ref_net_param_sizes(void* h, int layer, long long* nw, long long* nb) {
  RefNet* n = static_cast<RefNet*>(h);
  *nw = static_cast<long long>(n->states.layers[layer].weights.size());
  *nb = static_cast<long long>(n->states.layers[layer].bias.size());
}

void ref_net_get_params(void* h, int layer, float* w, float* b) {
  RefNet* n = static_cast<RefNet*>(h);
  const auto& st = n->states.layers[layer];
  if (w) std::memcpy(w, st.weights.data(), sizeof(float) * st.weights.size());
  if (b) std::memcpy(b, st.bias.data(), sizeof(float) * st.bias.size());
}

void ref_net_set_params(void* h, int layer, const float* w, const float* b) {
  RefNet* n = static_cast<RefNet*>(h);
  auto& st = n->states.layers[layer];
  if (w) std::memcpy(st.weights.data(), w, sizeof(float) * st.weights.size());
  if (b) std::memcpy(st.bias.data(), b, sizeof(float) * st.bias.size());
}

int ref_net_set_layer_fout(void* h, const char* layer, int f_out, double sigma) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    for (auto& l : n->spec.layers)
      if (l.name == layer) {
        l.f_out = f_out;
        if (l.init != InitKind::None && sigma > 0) l.init_sigma = sigma;
        return;
      }
    throw SpecError("no layer");
  });
}

int ref_net_output_extent(void* h, int w0, int* out) {
  return guard([&] { *out = output_extent(static_cast<RefNet*>(h)->spec, w0); });
}

long long ref_net_flops(void* h, int w0) {
  long long t = -1;
  guard([&] { t = flop_estimate(static_cast<RefNet*>(h)->spec, w0).total; });
  return t;
}

// Runs NetRunner<float>::forward (netgraph.hpp:64-84); output shape returned via c/hh/ww.
int ref_net_forward(void* h, const float* in, int C, int H, int W, int* oc, int* oh, int* ow) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    if (!n->runner) n->runner = std::make_unique<NetRunner<float>>(n->spec, n->states);
    const Blob<float> b = make_blob(in, C, H, W);
    n->last = n->runner->forward(b);
    *oc = n->last.channels;
    *oh = n->last.height;
    *ow = n->last.width;
  });
}

int ref_net_blob_shape(void* h, const char* name, int* c, int* hh, int* ww) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    if (!n->runner) throw SpecError("no runner");
    const Blob<float>& b = n->runner->blob(name);
    *c = b.channels;
    *hh = b.height;
    *ww = b.width;
  });
}

int ref_net_blob(void* h, const char* name, float* dst) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    if (!n->runner) throw SpecError("no runner");
    const Blob<float>& b = n->runner->blob(name);
    std::memcpy(dst, b.data.data(), sizeof(float) * b.size());
  });
}

// process<float> (pipeline.hpp:630-698): probs is C x H x W.
int ref_process(void* h, const uint8_t* img, int H, int W, int w, int v, uint8_t* labels,
                float* probs) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    Plane<std::uint8_t> p(H, W);
    std::memcpy(p.pix.data(), img, p.size());
    const ProcessResult<float> r = process(n->spec, n->states, p, w, v);
    std::memcpy(labels, r.labels.pix.data(), r.labels.size());
    for (std::size_t c = 0; c < r.probs.size(); ++c)
      std::memcpy(probs + c * static_cast<std::size_t>(H) * W, r.probs[c].pix.data(),
                  sizeof(float) * r.probs[c].size());
  });
}


// ---- file formats (fixtures for the CLI tests) ----
// save_weights (weights_io.hpp): the net's current parameters as a PXSG file.
int ref_save_weights(void* h, const char* path) {
  return guard([&] {
    RefNet* n = static_cast<RefNet*>(h);
    save_weights(path, n->spec, n->states);
  });
}

// write_pgm (image_io.hpp:83-93).
int ref_write_pgm(const char* path, const uint8_t* img, int H, int W) {
  return guard([&] {
    Plane<std::uint8_t> p(H, W);
    std::memcpy(p.pix.data(), img, p.size());
    write_pgm(path, p);
  });
}

// ---- training step ----
static NetRunner<float>& runner_of(RefNet* n) {
  if (!n->runner) throw SpecError("no runner (run forward first)");
  return *n->runner;
}

int ref_net_zero_blob_diffs(void* h) {
  return guard([&] { runner_of(static_cast<RefNet*>(h)).zero_blob_diffs(); });
}

// blob_mut(name).diff = src (the caller's seeding, netgraph.hpp:85-87)
int ref_net_set_blob_diff(void* h, const char* name, const float* src) {
  return guard([&] {
    Blob<float>& b = runner_of(static_cast<RefNet*>(h)).blob_mut(name);
    b.diff.assign(src, src + b.size());
  });
}

// Blob::diff of a blob (zeros when the diff is empty).
int ref_net_blob_diff(void* h, const char* name, float* dst) {
  return guard([&] {
    const Blob<float>& b = runner_of(static_cast<RefNet*>(h)).blob(name);
    if (b.diff.size() == b.size())
      std::memcpy(dst, b.diff.data(), sizeof(float) * b.size());
    else
      std::memset(dst, 0, sizeof(float) * b.size());
  });
}

int ref_net_backward(void* h) {
  return guard([&] { runner_of(static_cast<RefNet*>(h)).backward(); });
}

// which: 1 = weight_diff/bias_diff, 2 = weight_mom/bias_mom
void ref_net_param_state(void* h, int layer, int which, float* w, float* b) {
  const LayerState<float>& st = static_cast<RefNet*>(h)->states.layers[layer];
  const auto& vw = which == 1 ? st.weight_diff : st.weight_mom;
  const auto& vb = which == 1 ? st.bias_diff : st.bias_mom;
  if (w) std::memcpy(w, vw.data(), sizeof(float) * vw.size());
  if (b) std::memcpy(b, vb.data(), sizeof(float) * vb.size());
}

// softmax_loss (layers.hpp:269-307) on the runner's blob; mask may be NULL.
int ref_net_softmax_loss(void* h, const char* scores, const int* labels, const uint8_t* mask,
                         int H, int W, double* loss) {
  return guard([&] {
    Blob<float>& s = runner_of(static_cast<RefNet*>(h)).blob_mut(scores);
    Plane<int> lab(H, W);
    std::memcpy(lab.pix.data(), labels, sizeof(int) * lab.size());
    Plane<std::uint8_t> m;
    if (mask) {
      m = Plane<std::uint8_t>(H, W);
      std::memcpy(m.pix.data(), mask, m.size());
    }
    *loss = softmax_loss(s, lab, m);
  });
}

int ref_net_sgd_step(void* h, double lr, double momentum, double weight_decay) {
  return guard([&] {
    SolverConfig cfg;
    cfg.lr = lr;
    cfg.momentum = momentum;
    cfg.weight_decay = weight_decay;
    sgd_step(static_cast<RefNet*>(h)->states, cfg);
  });
}

// ---- layer-level backward functions (test_layers.cpp:107-389) ----
int ref_conv_backward_f32(const float* in, int C, int H, int W, const float* w, int f_out, int k, int d,
                          int s, int p, const float* dout, float* dw, float* db, float* din) {
  return guard([&] {
    Blob<float> x = make_blob(in, C, H, W);
    const ConvGeometry g = ConvGeometry::from_input(k, d, s, p, H, W);
    LayerState<float> st;
    st.init_conv(f_out, C * k * k);
    std::memcpy(st.weights.data(), w, sizeof(float) * st.weights.size());
    std::memcpy(st.weight_diff.data(), dw, sizeof(float) * st.weight_diff.size());
    std::memcpy(st.bias_diff.data(), db, sizeof(float) * st.bias_diff.size());
    if (din) x.diff.assign(din, din + x.size());
    Blob<float> out(f_out, g.out_h, g.out_w);
    out.diff.assign(dout, dout + out.size());
    ColumnBuffer<float> cb, cg;
    conv_sk_backward(x, st, f_out, g, cb, cg, out, din != nullptr);
    std::memcpy(dw, st.weight_diff.data(), sizeof(float) * st.weight_diff.size());
    std::memcpy(db, st.bias_diff.data(), sizeof(float) * st.bias_diff.size());
    if (din) std::memcpy(din, x.diff.data(), sizeof(float) * x.size());
  });
}

int ref_col2im_f32(const float* col, int C, int H, int W, int k, int d, int s, int p, float* out) {
  return guard([&] {
    const ConvGeometry g = ConvGeometry::from_input(k, d, s, p, H, W);
    ColumnBuffer<float> cb;
    cb.resize(C * k * k, g.out_h * g.out_w);
    std::memcpy(cb.data.data(), col, sizeof(float) * cb.rows * cb.cols);
    Blob<float> o;
    col2im_sk(cb, g, C, o);
    std::memcpy(out, o.data.data(), sizeof(float) * o.size());
  });
}

int ref_maxpool_backward_f32(const uint64_t* argmax, const float* dout, int n_out, int C, int H, int W,
                             float* din) {
  return guard([&] {
    Blob<float> x(C, H, W);
    x.diff.assign(din, din + x.size());
    LayerState<float> st;
    st.argmax.assign(argmax, argmax + n_out);
    Blob<float> out(1, 1, n_out);
    out.diff.assign(dout, dout + n_out);
    maxpool_sk_backward(x, st, out);
    std::memcpy(din, x.diff.data(), sizeof(float) * x.size());
  });
}

void ref_relu_backward_f32(const float* in, const float* dout, int n, float* din) {
  Blob<float> x(1, 1, n), out(1, 1, n);
  std::memcpy(x.data.data(), in, sizeof(float) * n);
  x.diff.assign(din, din + n);
  out.diff.assign(dout, dout + n);
  relu_backward(x, out);
  std::memcpy(din, x.diff.data(), sizeof(float) * n);
}

void ref_upconv_backward_f32(const float* dout, int C, int H, int W, float* din) {
  Blob<float> x(C, H, W), out(C, 2 * H, 2 * W);
  x.diff.assign(din, din + x.size());
  out.diff.assign(dout, dout + out.size());
  upconv_backward(x, out);
  std::memcpy(din, x.diff.data(), sizeof(float) * x.size());
}

void ref_mergecrop_backward_f32(const float* dout, int Ca, int Cb, int H, int W, float* da) {
  Blob<float> a(Ca, H, W), out(Ca + Cb, H, W);
  a.diff.assign(da, da + a.size());
  out.diff.assign(dout, dout + out.size());
  mergecrop_backward(a, out);
  std::memcpy(da, a.diff.data(), sizeof(float) * a.size());
}

void ref_softmax_backward_f32(const float* out_data, const float* dout, int C, int H, int W, float* din) {
  Blob<float> x(C, H, W), out(C, H, W);
  std::memcpy(out.data.data(), out_data, sizeof(float) * out.size());
  out.diff.assign(dout, dout + out.size());
  x.diff.assign(din, din + x.size());
  softmax_backward(x, out);
  std::memcpy(din, x.diff.data(), sizeof(float) * x.size());
}

int ref_softmax_loss_f32(const float* scores, int C, int H, int W, const int* labels, const uint8_t* mask,
                         float* dscores, double* loss) {
  return guard([&] {
    Blob<float> s = make_blob(scores, C, H, W);
    s.diff.assign(dscores, dscores + s.size());
    Plane<int> lab(H, W);
    std::memcpy(lab.pix.data(), labels, sizeof(int) * lab.size());
    Plane<std::uint8_t> m;
    if (mask) {
      m = Plane<std::uint8_t>(H, W);
      std::memcpy(m.pix.data(), mask, m.size());
    }
    *loss = softmax_loss(s, lab, m);
    if (s.diff.size() == s.size()) std::memcpy(dscores, s.diff.data(), sizeof(float) * s.size());
  });
}

void ref_sgd_step_f32(float* w, float* mom, float* diff, int n, double lr, double momentum, double wd) {
  NetStates<float> st;
  st.layers.resize(1);
  st.layers[0].weights.assign(w, w + n);
  st.layers[0].weight_mom.assign(mom, mom + n);
  st.layers[0].weight_diff.assign(diff, diff + n);
  SolverConfig cfg;
  cfg.lr = lr;
  cfg.momentum = momentum;
  cfg.weight_decay = wd;
  sgd_step(st, cfg);
  std::memcpy(w, st.layers[0].weights.data(), sizeof(float) * n);
  std::memcpy(mom, st.layers[0].weight_mom.data(), sizeof(float) * n);
  std::memcpy(diff, st.layers[0].weight_diff.data(), sizeof(float) * n);
}

// ---- MALIS (malis.hpp): affinity graph, components, maximin gradient, composed loss --------
}  // extern "C"

namespace {
template <typename S>
Plane<S> plane_of(const S* p, int h, int w) {
  Plane<S> q(h, w);
  std::memcpy(q.pix.data(), p, sizeof(S) * q.size());
  return q;
}
template <typename S>
void ref_affinity_forward(const S* fg, int h, int w, S* a_x, S* a_y, uint8_t* m_x, uint8_t* m_y) {
  const AffinityGraph<S> g = affinity_forward(plane_of(fg, h, w));
  std::memcpy(a_x, g.a_x.pix.data(), sizeof(S) * g.a_x.size());
  std::memcpy(a_y, g.a_y.pix.data(), sizeof(S) * g.a_y.size());
  std::memcpy(m_x, g.m_x.pix.data(), g.m_x.size());
  std::memcpy(m_y, g.m_y.pix.data(), g.m_y.size());
}
template <typename S>
int ref_affinity_backward(const S* da_x, const S* da_y, const uint8_t* m_x, const uint8_t* m_y, int h, int w,
                          S* d_pos, S* d_neg) {
  return guard([&] {
    AffinityGraph<S> g(h, w);
    std::memcpy(g.m_x.pix.data(), m_x, g.m_x.size());
    std::memcpy(g.m_y.pix.data(), m_y, g.m_y.size());
    Plane<S> dp, dn;
    affinity_backward(plane_of(da_x, h, w), plane_of(da_y, h, w), g, dp, dn);
    std::memcpy(d_pos, dp.pix.data(), sizeof(S) * dp.size());
    std::memcpy(d_neg, dn.pix.data(), sizeof(S) * dn.size());
  });
}
template <typename S>
int ref_malis_gradient(const S* p_ax, const S* p_ay, const S* t_ax, const S* t_ay, const int* comp, int h, int w,
                       S* da_x, S* da_y, long long* pos_x, long long* pos_y, long long* neg_x, long long* neg_y,
                       long long* totals, double* losses) {
  return guard([&] {
    AffinityGraph<S> pred(h, w), truth(h, w);
    pred.a_x = plane_of(p_ax, h, w);
    pred.a_y = plane_of(p_ay, h, w);
    truth.a_x = plane_of(t_ax, h, w);
    truth.a_y = plane_of(t_ay, h, w);
    const MalisResult<S> r = malis_gradient(pred, truth, plane_of(comp, h, w));
    const size_t n = static_cast<size_t>(h) * w;
    std::memcpy(da_x, r.da_x.pix.data(), sizeof(S) * n);
    std::memcpy(da_y, r.da_y.pix.data(), sizeof(S) * n);
    std::memcpy(pos_x, r.pos_x.pix.data(), sizeof(long long) * n);
    std::memcpy(pos_y, r.pos_y.pix.data(), sizeof(long long) * n);
    std::memcpy(neg_x, r.neg_x.pix.data(), sizeof(long long) * n);
    std::memcpy(neg_y, r.neg_y.pix.data(), sizeof(long long) * n);
    totals[0] = r.total_pos;
    totals[1] = r.total_neg;
    losses[0] = r.loss_pos;
    losses[1] = r.loss_neg;
    losses[2] = r.loss;
  });
}
template <typename S>
int ref_malis_softmax_loss(const S* scores, int C, int h, int w, const uint8_t* fg, S* diff, double* loss) {
  return guard([&] {
    Blob<S> s = make_blob(scores, C, h, w);
    s.diff.assign(diff, diff + s.size());
    *loss = malis_softmax_loss(s, plane_of(fg, h, w));
    std::memcpy(diff, s.diff.data(), sizeof(S) * s.size());
  });
}
}  // namespace

extern "C" {
void ref_affinity_forward_f32(const float* fg, int h, int w, float* ax, float* ay, uint8_t* mx, uint8_t* my) {
  ref_affinity_forward(fg, h, w, ax, ay, mx, my);
}
void ref_affinity_forward_f64(const double* fg, int h, int w, double* ax, double* ay, uint8_t* mx, uint8_t* my) {
  ref_affinity_forward(fg, h, w, ax, ay, mx, my);
}
int ref_affinity_backward_f32(const float* dax, const float* day, const uint8_t* mx, const uint8_t* my, int h,
                              int w, float* dp, float* dn) {
  return ref_affinity_backward(dax, day, mx, my, h, w, dp, dn);
}
int ref_affinity_backward_f64(const double* dax, const double* day, const uint8_t* mx, const uint8_t* my, int h,
                              int w, double* dp, double* dn) {
  return ref_affinity_backward(dax, day, mx, my, h, w, dp, dn);
}
void ref_connected_components(const uint8_t* labels, int h, int w, int* comp) {
  const Plane<int> c = connected_components(plane_of(labels, h, w));
  std::memcpy(comp, c.pix.data(), sizeof(int) * c.size());
}
int ref_malis_gradient_f32(const float* pax, const float* pay, const float* tax, const float* tay, const int* comp,
                           int h, int w, float* dax, float* day, long long* px, long long* py, long long* nx,
                           long long* ny, long long* totals, double* losses) {
  return ref_malis_gradient(pax, pay, tax, tay, comp, h, w, dax, day, px, py, nx, ny, totals, losses);
}
int ref_malis_gradient_f64(const double* pax, const double* pay, const double* tax, const double* tay,
                           const int* comp, int h, int w, double* dax, double* day, long long* px, long long* py,
                           long long* nx, long long* ny, long long* totals, double* losses) {
  return ref_malis_gradient(pax, pay, tax, tay, comp, h, w, dax, day, px, py, nx, ny, totals, losses);
}
int ref_malis_softmax_loss_f32(const float* scores, int C, int h, int w, const uint8_t* fg, float* diff,
                               double* loss) {
  return ref_malis_softmax_loss(scores, C, h, w, fg, diff, loss);
}
int ref_malis_softmax_loss_f64(const double* scores, int C, int h, int w, const uint8_t* fg, double* diff,
                               double* loss) {
  return ref_malis_softmax_loss(scores, C, h, w, fg, diff, loss);
}
}  // extern "C"
