// test_dropin.cpp -- the C++ drop-in (include/pixelseg_gpu.hpp) against the reference itself,
// both compiled into one binary: every check compares pixelseg::gpu::X with pixelseg::X on the
// same inputs, bit for bit. Built by __graft_entry__.build() where /root/reference exists (the
// reference headers are compile-time only); run on the B200 by tests/test_gpu_dropin_cpp.py.
// Cases follow proj/tests/test_layers.cpp, test_netgraph.cpp and test_pipeline.cpp.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pixelseg_gpu.hpp"

using namespace pixelseg;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, what)                                               \
  do {                                                                  \
    if (cond) {                                                         \
      ++g_pass;                                                         \
    } else {                                                            \
      ++g_fail;                                                         \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__);       \
    }                                                                   \
  } while (0)

template <typename T>
static bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0;
}

template <typename S>
static void fill(std::vector<S>& v, Rng& r) {
  for (auto& x : v) x = static_cast<S>(r.uniform(-1.0, 1.0));
}

template <typename S>
static void conv_cases() {
  Rng rng(5);
  struct Case { int f_in, f_out, h, w, k, d, s, p; };
  const Case cases[] = {{3, 4, 9, 9, 3, 1, 1, 0}, {2, 5, 11, 11, 3, 2, 1, 0}, {4, 2, 8, 8, 2, 1, 2, 0},
                        {1, 3, 7, 7, 7, 1, 1, 0}, {2, 2, 6, 6, 3, 1, 1, 1}, {12, 130, 40, 40, 10, 3, 1, 0}};
  for (const auto& c : cases) {
    Blob<S> in(c.f_in, c.h, c.w);
    fill(in.data, rng);
    LayerState<S> st;
    st.init_conv(c.f_out, c.f_in * c.k * c.k);
    fill(st.weights, rng);
    fill(st.bias, rng);
    const ConvGeometry g = ConvGeometry::from_input(c.k, c.d, c.s, c.p, c.h, c.w);
    ColumnBuffer<S> cb;
    Blob<S> ref, got;
    conv_sk_forward(in, st, c.f_out, g, cb, ref);
    gpu::conv_sk_forward(in, st, c.f_out, g, cb, got);
    CHECK(same_bits(ref.data, got.data), "conv_sk_forward");
    CHECK(got.channels == ref.channels && got.height == ref.height, "conv shape");
  }
}

static void layer_cases() {
  Rng rng(11);
  for (int t = 0; t < 3; ++t) {
    const int k = 2, d = t + 1, s = t == 0 ? 2 : 1, hw = 10 + t;
    Blob<float> in(3, hw, hw);
    fill(in.data, rng);
    const ConvGeometry g = ConvGeometry::from_input(k, d, s, 0, hw, hw);
    LayerState<float> s1, s2;
    Blob<float> a, b;
    maxpool_sk_forward(in, s1, g, a);
    gpu::maxpool_sk_forward(in, s2, g, b);
    CHECK(same_bits(a.data, b.data) && s1.argmax == s2.argmax, "maxpool_sk_forward");
    relu_forward(in, a);
    gpu::relu_forward(in, b);
    CHECK(same_bits(a.data, b.data), "relu_forward");
    upconv_forward(in, a);
    gpu::upconv_forward(in, b);
    CHECK(same_bits(a.data, b.data), "upconv_forward");
    softmax_forward(in, a);
    gpu::softmax_forward(in, b);
    CHECK(same_bits(a.data, b.data), "softmax_forward");
    Blob<float> small(2, hw - 3, hw - 4);
    fill(small.data, rng);
    mergecrop_forward(small, in, a);
    gpu::mergecrop_forward(small, in, b);
    CHECK(same_bits(a.data, b.data), "mergecrop_forward");
    ColumnBuffer<float> c1, c2;
    const ConvGeometry gc = ConvGeometry::from_input(3, d, 1, 1, hw, hw);
    im2col_sk(in, gc, c1);
    gpu::im2col_sk(in, gc, c2);
    c1.data.resize(static_cast<std::size_t>(c1.rows) * c1.cols);
    c2.data.resize(static_cast<std::size_t>(c2.rows) * c2.cols);
    CHECK(same_bits(c1.data, c2.data), "im2col_sk");
  }
  // gemm, all transposes, alpha/beta
  const int m = 7, n = 9, kk = 13;
  std::vector<float> A(m * kk), B(kk * n), C0(m * n);
  fill(A, rng);
  fill(B, rng);
  fill(C0, rng);
  for (int ta = 0; ta < 2; ++ta)
    for (int tb = 0; tb < 2; ++tb) {
      std::vector<float> c1 = C0, c2 = C0;
      gemm<float>(ta, tb, m, n, kk, 0.5f, A.data(), B.data(), 1.5f, c1.data());
      gpu::gemm<float>(ta, tb, m, n, kk, 0.5f, A.data(), B.data(), 1.5f, c2.data());
      CHECK(same_bits(c1, c2), "gemm");
    }
  // errors: same types and messages
  LayerState<float> st;
  st.init_conv(3, 2 * 9);
  ColumnBuffer<float> cb;
  Blob<float> in(2, 5, 5), out;
  std::string e1, e2;
  try { conv_sk_forward(in, st, 3, ConvGeometry::from_input(5, 1, 1, 0, 5, 5), cb, out); } catch (const SizeError& e) { e1 = e.what(); }
  try { gpu::conv_sk_forward(in, st, 3, ConvGeometry::from_input(5, 1, 1, 0, 5, 5), cb, out); } catch (const SizeError& e) { e2 = e.what(); }
  CHECK(!e1.empty() && e1 == e2, "conv weight-count error");
}

static void net_cases() {
  const NetSpec spec = parse_netspec_or_throw(
      "input w=8 f=2\n"
      "layer conv1 conv_sk k=3 fout=3 in=data out=conv1 init=gaussian:0.5\n"
      "layer relu1 relu in=conv1 out=relu1\n"
      "layer pool1 pool_max k=2 s=2 in=relu1 out=pool1\n"
      "layer conv2 conv_sk k=3 fout=2 in=pool1 out=conv2 init=gaussian:0.5\n"
      "layer prob softmax_loss in=conv2 out=prob\n");
  auto states = init_weights<float>(spec, 7);
  Blob<float> input(2, 8, 8);
  Rng rng(99);
  fill(input.data, rng);
  NetRunner<float> ref(spec, states);
  gpu::NetRunner<float> got(spec, states);
  const Blob<float> r = ref.forward(input);
  const Blob<float> g = got.forward(input);
  CHECK(same_bits(r.data, g.data), "NetRunner::forward");
  for (const char* name : {"conv1", "relu1", "pool1", "conv2"})
    CHECK(same_bits(ref.blob(name).data, got.blob(name).data), name);
  // weights change between calls -> the drop-in re-uploads
  states.layers[1].weights[0] += 0.25f;
  CHECK(same_bits(ref.forward(input).data, got.forward(input).data), "forward after weight change");
  std::string e1, e2;
  try { ref.forward(Blob<float>(3, 8, 8)); } catch (const SizeError& e) { e1 = e.what(); }
  try { got.forward(Blob<float>(3, 8, 8)); } catch (const SizeError& e) { e2 = e.what(); }
  CHECK(!e1.empty() && e1 == e2, "forward channel error");
  try { ref.forward(Blob<float>(2, 2, 2)); } catch (const SizeError& e) { e1 = e.what(); }
  try { got.forward(Blob<float>(2, 2, 2)); } catch (const SizeError& e) { e2 = e.what(); }
  CHECK(e1 == e2, "forward layer error");
}

static void process_cases() {
  const NetSpec spec = parse_netspec_or_throw(
      "input w=21 f=1\n"
      "layer c1 conv_sk k=3 fout=4 in=data out=c1 init=he\n"
      "layer r1 relu in=c1 out=r1\n"
      "layer p1 pool_max k=2 s=1 in=r1 out=p1\n"
      "layer c2 conv_sk k=2 d=2 fout=3 in=p1 out=c2 init=he\n"
      "layer prob softmax_loss in=c2 out=prob\n");
  NetStates<float> states = init_weights<float>(spec, 17);
  Rng rng(55);
  Plane<std::uint8_t> img(37, 29);
  for (auto& p : img.pix) p = static_cast<std::uint8_t>(rng.uniform_index(256));
  for (int w : {16, 8, 5}) {
    const ProcessResult<float> a = process(spec, states, img, w, 5);
    const ProcessResult<float> b = gpu::process(spec, states, img, w, 5);
    CHECK(a.labels.pix == b.labels.pix, "process labels");
    bool ok = a.probs.size() == b.probs.size();
    for (std::size_t c = 0; ok && c < a.probs.size(); ++c) ok = same_bits(a.probs[c].pix, b.probs[c].pix);
    CHECK(ok, "process probs");
  }
  std::string e1, e2;
  try { process(spec, states, img, 16, 4); } catch (const SpecError& e) { e1 = e.what(); }
  try { gpu::process(spec, states, img, 16, 4); } catch (const SpecError& e) { e2 = e.what(); }
  CHECK(!e1.empty() && e1 == e2, "process tile error");
}

// Training step: reference NetRunner::backward / softmax_loss / sgd_step
// vs the drop-ins, two SGD iterations, plus a diff seeded through blob_mut (test_netgraph.cpp).
static void train_cases() {
  const char* texts[] = {
      "input w=12 f=2\n"
      "layer conv1 conv_sk k=3 fout=4 in=data out=conv1 init=gaussian:0.5\n"
      "layer relu1 relu in=conv1 out=relu1\n"
      "layer pool1 pool_max k=2 s=2 in=relu1 out=pool1\n"
      "layer conv2 conv_sk k=3 fout=3 in=pool1 out=conv2 init=gaussian:0.5\n"
      "layer prob softmax_loss in=conv2 out=prob\n",
      "input w=16 f=1\n"
      "layer conv1 conv_sk k=3 fout=2 in=data out=conv1 init=gaussian:0.4\n"
      "layer pool1 pool_max k=2 s=2 in=conv1 out=pool1\n"
      "layer conv2 conv_sk k=3 fout=4 in=pool1 out=conv2 init=gaussian:0.4\n"
      "layer up1 upconv in=conv2 out=up1\n"
      "layer merge1 mergecrop in=up1,conv1 out=merge1\n"
      "layer conv3 conv_sk k=3 d=2 fout=2 in=merge1 out=conv3 init=gaussian:0.4\n"
      "layer prob softmax_loss in=conv3 out=prob\n"};
  for (const char* text : texts) {
    const NetSpec spec = parse_netspec_or_throw(text);
    NetStates<float> s_ref = init_weights<float>(spec, 7), s_gpu = init_weights<float>(spec, 7);
    NetRunner<float> ref(spec, s_ref);
    gpu::NetRunner<float> got(spec, s_gpu);
    SolverConfig cfg;
    cfg.lr = 0.05;
    cfg.momentum = 0.9;
    cfg.weight_decay = 5e-4;
    Rng rng(3);
    const std::string scores = spec.layers.back().inputs[0];
    for (int it = 0; it < 2; ++it) {
      Blob<float> x(spec.f0, spec.w0, spec.w0);
      fill(x.data, rng);
      const Blob<float>& o1 = ref.forward(x);
      const Blob<float>& o2 = got.forward(x);
      CHECK(same_bits(o1.data, o2.data), "train forward");
      ref.zero_blob_diffs();
      got.zero_blob_diffs();
      Plane<int> lab(o1.height, o1.width);
      for (auto& v : lab.pix) v = static_cast<int>(rng.uniform_index(o1.channels));
      Plane<std::uint8_t> mask(o1.height, o1.width, 1);
      for (auto& v : mask.pix) v = rng.coin() ? 1 : 0;
      const double l1 = softmax_loss(ref.blob_mut(scores), lab, mask);
      const double l2 = gpu::softmax_loss(got, scores, lab, mask);
      CHECK(std::memcmp(&l1, &l2, sizeof l1) == 0, "softmax_loss");
      ref.backward();
      got.backward();
      for (const auto& l : spec.layers)
        CHECK(same_bits(ref.blob(l.output).diff, got.blob_mut(l.output).diff), "backward blob diff");
      for (std::size_t i = 0; i < spec.layers.size(); ++i) {
        CHECK(same_bits(s_ref.layers[i].weight_diff, s_gpu.layers[i].weight_diff), "weight_diff");
        CHECK(same_bits(s_ref.layers[i].bias_diff, s_gpu.layers[i].bias_diff), "bias_diff");
      }
      sgd_step(s_ref, cfg);
      gpu::sgd_step(got, cfg);
      for (std::size_t i = 0; i < spec.layers.size(); ++i) {
        CHECK(same_bits(s_ref.layers[i].weights, s_gpu.layers[i].weights), "sgd weights");
        CHECK(same_bits(s_ref.layers[i].bias, s_gpu.layers[i].bias), "sgd bias");
        CHECK(same_bits(s_ref.layers[i].weight_mom, s_gpu.layers[i].weight_mom), "sgd momentum");
      }
    }
    // a diff seeded at the probability blob (softmax_backward)
    Blob<float> x(spec.f0, spec.w0, spec.w0);
    fill(x.data, rng);
    ref.forward(x);
    got.forward(x);
    const std::string prob = spec.layers.back().output;
    std::vector<float> seed(ref.blob(prob).size());
    fill(seed, rng);
    ref.blob_mut(prob).diff = seed;
    got.blob_mut(prob).diff = seed;
    ref.backward();
    got.backward();
    for (const auto& l : spec.layers)
      CHECK(same_bits(ref.blob(l.output).diff, got.blob_mut(l.output).diff), "seeded backward diff");
  }
}

// Layer-level backward functions (test_layers.cpp:107-389) vs the drop-ins.
static void backward_layer_cases() {
  Rng rng(41);
  struct Case { int f_in, f_out, h, w, k, d, s, p; };
  const Case cases[] = {{3, 4, 9, 9, 3, 1, 1, 0}, {2, 5, 11, 11, 3, 2, 1, 0}, {4, 2, 8, 8, 2, 1, 2, 0},
                        {2, 2, 6, 6, 3, 1, 1, 1}, {12, 130, 40, 40, 10, 3, 1, 0}};
  for (const auto& c : cases) {
    const ConvGeometry g = ConvGeometry::from_input(c.k, c.d, c.s, c.p, c.h, c.w);
    Blob<float> in1(c.f_in, c.h, c.w);
    fill(in1.data, rng);
    in1.ensure_diff();
    fill(in1.diff, rng);
    Blob<float> in2 = in1;
    LayerState<float> s1;
    s1.init_conv(c.f_out, c.f_in * c.k * c.k);
    fill(s1.weights, rng);
    fill(s1.weight_diff, rng);
    fill(s1.bias_diff, rng);
    LayerState<float> s2 = s1;
    Blob<float> out(c.f_out, g.out_h, g.out_w);
    out.ensure_diff();
    fill(out.diff, rng);
    ColumnBuffer<float> cb, cg;
    conv_sk_backward(in1, s1, c.f_out, g, cb, cg, out, true);
    gpu::conv_sk_backward(in2, s2, c.f_out, g, cb, cg, out, true);
    CHECK(same_bits(s1.weight_diff, s2.weight_diff), "conv_sk_backward dW");
    CHECK(same_bits(s1.bias_diff, s2.bias_diff), "conv_sk_backward db");
    CHECK(same_bits(in1.diff, in2.diff), "conv_sk_backward din");
    ColumnBuffer<float> col;
    col.resize(c.f_in * c.k * c.k, g.out_h * g.out_w);
    fill(col.data, rng);
    Blob<float> o1, o2;
    col2im_sk(col, g, c.f_in, o1);
    gpu::col2im_sk(col, g, c.f_in, o2);
    CHECK(same_bits(o1.data, o2.data), "col2im_sk");
  }
  {  // pooling with ties, then backward through the argmax
    Blob<float> x(3, 13, 13);
    for (auto& v : x.data) v = static_cast<float>(static_cast<int>(rng.uniform(0.0, 4.0))) * 0.5f;
    const ConvGeometry g = ConvGeometry::from_input(2, 2, 1, 0, 13, 13);
    LayerState<float> st;
    Blob<float> y;
    maxpool_sk_forward(x, st, g, y);
    y.ensure_diff();
    fill(y.diff, rng);
    Blob<float> a = x, b = x;
    a.ensure_diff();
    fill(a.diff, rng);
    b.diff = a.diff;
    maxpool_sk_backward(a, st, y);
    gpu::maxpool_sk_backward(b, st, y);
    CHECK(same_bits(a.diff, b.diff), "maxpool_sk_backward");
    Blob<float> r1 = x, r2 = x, ro(3, 13, 13);
    ro.ensure_diff();
    fill(ro.diff, rng);
    relu_backward(r1, ro);
    gpu::relu_backward(r2, ro);
    CHECK(same_bits(r1.diff, r2.diff), "relu_backward");
    Blob<float> u1(3, 6, 7), u2(3, 6, 7), uo(3, 12, 14);
    uo.ensure_diff();
    fill(uo.diff, rng);
    upconv_backward(u1, uo);
    gpu::upconv_backward(u2, uo);
    CHECK(same_bits(u1.diff, u2.diff), "upconv_backward");
    Blob<float> m1(2, 5, 5), m2(2, 5, 5), mo(5, 5, 5);
    mo.ensure_diff();
    fill(mo.diff, rng);
    mergecrop_backward(m1, mo);
    gpu::mergecrop_backward(m2, mo);
    CHECK(same_bits(m1.diff, m2.diff), "mergecrop_backward");
    Blob<float> sc(3, 4, 5), pr;
    fill(sc.data, rng);
    softmax_forward(sc, pr);
    pr.ensure_diff();
    fill(pr.diff, rng);
    Blob<float> s1 = sc, s2 = sc;
    softmax_backward(s1, pr);
    gpu::softmax_backward(s2, pr);
    CHECK(same_bits(s1.diff, s2.diff), "softmax_backward");
    Plane<int> lab(4, 5);
    for (auto& v : lab.pix) v = static_cast<int>(rng.uniform_index(3));
    Plane<std::uint8_t> mask(4, 5, 1);
    Blob<float> l1 = sc, l2 = sc;
    const double a1 = softmax_loss(l1, lab, mask), a2 = gpu::softmax_loss(l2, lab, mask);
    CHECK(std::memcmp(&a1, &a2, sizeof a1) == 0 && same_bits(l1.diff, l2.diff), "softmax_loss (layer)");
  }
  {  // sgd_step over NetStates (test_pipeline.cpp:336-395)
    const NetSpec spec = parse_netspec_or_throw(
        "input w=8 f=1\nlayer c1 conv_sk k=3 fout=4 in=data out=c1 init=he\n"
        "layer prob softmax_loss in=c1 out=prob\n");
    NetStates<float> a = init_weights<float>(spec, 5);
    for (auto& st : a.layers) {
      fill(st.weight_diff, rng);
      fill(st.weight_mom, rng);
      fill(st.bias_diff, rng);
    }
    NetStates<float> b = a;
    SolverConfig cfg;
    cfg.lr = 0.03;
    cfg.momentum = 0.8;
    cfg.weight_decay = 1e-3;
    sgd_step(a, cfg);
    gpu::sgd_step(b, cfg);
    for (std::size_t i = 0; i < a.layers.size(); ++i) {
      CHECK(same_bits(a.layers[i].weights, b.layers[i].weights), "sgd_step weights");
      CHECK(same_bits(a.layers[i].weight_mom, b.layers[i].weight_mom), "sgd_step momentum");
      CHECK(same_bits(a.layers[i].weight_diff, b.layers[i].weight_diff), "sgd_step diff");
      CHECK(same_bits(a.layers[i].bias, b.layers[i].bias), "sgd_step bias");
    }
  }
}

// MALIS (malis.hpp) vs proj/tests/test_malis.cpp-style random instances, both S.
template <typename S>
static void malis_cases() {
  Rng rng(909);
  for (int trial = 0; trial < 12; ++trial) {
    const int h = 1 + static_cast<int>(rng.uniform_index(20)), w = 1 + static_cast<int>(rng.uniform_index(20));
    Plane<std::uint8_t> fg(h, w);
    for (auto& v : fg.pix) v = rng.coin() ? 1 : 0;
    Plane<S> probs(h, w), fgt(h, w);
    for (auto& v : probs.pix) v = static_cast<S>(rng.uniform(0.01, 0.99));
    for (std::size_t i = 0; i < fg.size(); ++i) fgt.pix[i] = fg.pix[i] ? S(1) : S(0);
    const auto pr = affinity_forward(probs), pg = gpu::affinity_forward(probs);
    CHECK(same_bits(pr.a_x.pix, pg.a_x.pix) && same_bits(pr.a_y.pix, pg.a_y.pix) &&
              same_bits(pr.m_x.pix, pg.m_x.pix) && same_bits(pr.m_y.pix, pg.m_y.pix),
          "affinity_forward");
    const auto tr = affinity_forward(fgt);
    const Plane<int> cr = connected_components(fg), cg = gpu::connected_components(fg);
    CHECK(same_bits(cr.pix, cg.pix), "connected_components");
    const auto rr = malis_gradient(pr, tr, cr);
    const auto rg = gpu::malis_gradient(pr, tr, cr);
    CHECK(same_bits(rr.da_x.pix, rg.da_x.pix) && same_bits(rr.da_y.pix, rg.da_y.pix), "malis_gradient da");
    CHECK(same_bits(rr.pos_x.pix, rg.pos_x.pix) && same_bits(rr.pos_y.pix, rg.pos_y.pix) &&
              same_bits(rr.neg_x.pix, rg.neg_x.pix) && same_bits(rr.neg_y.pix, rg.neg_y.pix),
          "malis_gradient pair counts");
    CHECK(rr.total_pos == rg.total_pos && rr.total_neg == rg.total_neg && rr.loss == rg.loss &&
              rr.loss_pos == rg.loss_pos && rr.loss_neg == rg.loss_neg,
          "malis_gradient totals and losses");
    Plane<S> dpr, dnr, dpg, dng;
    affinity_backward(rr.da_x, rr.da_y, pr, dpr, dnr);
    gpu::affinity_backward(rr.da_x, rr.da_y, pr, dpg, dng);
    CHECK(same_bits(dpr.pix, dpg.pix) && same_bits(dnr.pix, dng.pix), "affinity_backward");
    Blob<S> sr(2, h, w);
    fill(sr.data, rng);
    sr.ensure_diff();
    fill(sr.diff, rng);
    Blob<S> sg = sr;
    const double lr = malis_softmax_loss(sr, fg), lg = gpu::malis_softmax_loss(sg, fg);
    CHECK(lr == lg && same_bits(sr.diff, sg.diff), "malis_softmax_loss");
  }
  Blob<S> three(3, 2, 2);
  Plane<std::uint8_t> fg(2, 2, 1);
  std::string msg;
  try {
    gpu::malis_softmax_loss(three, fg);
  } catch (const SizeError& e) {
    msg = e.what();
  }
  CHECK(msg == "malis loss: needs exactly 2 score channels, got 3", "malis loss channel check");
}

int main() {
  malis_cases<float>();
  malis_cases<double>();
  train_cases();
  backward_layer_cases();
  conv_cases<float>();
  conv_cases<double>();
  layer_cases();
  net_cases();
  process_cases();
  std::printf("drop-in vs reference: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
