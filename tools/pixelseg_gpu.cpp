// pixelseg_gpu -- the reference CLI's GPU-path subcommands (proj/tools/pixelseg.cpp) on the
// B200 drop-ins of include/pixelseg_gpu.hpp.
//
//   process --net N --weights W --in IMG --out DIR [--prob] [--tile T] [--gpus G]
//                                                                        (pixelseg.cpp:161-191)
//   bench   --net N [--w0 W] [--trials T] [--peak-gflops P] [--seed S] [--backward]
//                                                                        (pixelseg.cpp:193-267)
//   sizes   --net N [--w0 W]                                             (pixelseg.cpp:97-101)
//   flops   --net N [--w0 W]                                             (pixelseg.cpp:113-121)
//
// Same inputs (net spec text, PXSG weights, PGM/PNG images: the reference's own netspec.hpp,
// weights_io.hpp and image_io.hpp, which a caller keeps), same stdout lines, same output files
// and the same exit codes (0 ok, 1 usage, 2 spec/geometry, 3 I/O, 4 numeric; pixelseg.cpp:4-5,
// :465-475). The only change against the reference tool is that process() and NetRunner are
// pixelseg::gpu:: -- labels and probability maps are bit-identical.
//
// The reference parses its flags with CLI11 (absent here); this file parses the same flag
// names by hand. `--gpus G` (process) is the one addition: tile-row bands on G GPUs of this
// node (pixelseg::gpu::process(..., n_gpus), graft_multi_process), the same output files.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "pixelseg/convert.hpp"
#include "pixelseg/image_io.hpp"
#include "pixelseg/netgraph.hpp"
#include "pixelseg/netspec.hpp"
#include "pixelseg/pipeline.hpp"
#include "pixelseg/rng.hpp"
#include "pixelseg/weights_io.hpp"
#include "pixelseg_gpu.hpp"

using namespace pixelseg;

namespace {

struct Usage {
  std::string msg;
};

NetSpec load_net(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f.good()) throw IoError("cannot open '" + path + "' for reading");
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const ParseResult parsed = parse_netspec(text);
  if (!parsed.ok()) throw SpecError("'" + path + "':\n" + parsed.issue_text());
  return parsed.spec;
}

// "%.6g", the reference tool's number format for timings and rates.
std::string g6(double x) {
  char b[48];
  std::snprintf(b, sizeof b, "%.6g", x);
  return b;
}

// Tab-separated "a<TAB>b<TAB>c" output row.
template <typename... T>
void row(const T&... cols) {
  const char* sep = "";
  ((std::cout << sep << cols, sep = "\t"), ...);
  std::cout << "\n";
}

double median_of(std::vector<double> xs) {
  if (xs.empty()) return 0.0;
  const std::size_t h = xs.size() / 2;
  std::nth_element(xs.begin(), xs.begin() + h, xs.end());
  if (xs.size() & 1) return xs[h];
  const double hi = xs[h];
  return 0.5 * (*std::max_element(xs.begin(), xs.begin() + h) + hi);
}

int cmd_sizes(const NetSpec& spec, int w0) {
  const SizeTable t = propagate_sizes(spec, w0 > 0 ? w0 : spec.w0);
  std::cout << "# layer\tkind\tk\ts\td\tf_in\tf_out\tw_in\tw_out\n";
  for (const auto& r : t) row(r.name, kind_name(r.kind), r.k, r.s, r.d, r.f_in, r.f_out, r.w_in, r.w_out);
  if (!t.empty()) std::cout << "# output extent: " << t.back().w_out << "\n";
  return 0;
}

int cmd_flops(const NetSpec& spec, int w0) {
  const int w = w0 > 0 ? w0 : spec.w0;
  const FlopTable t = flop_estimate(spec, w);
  std::cout << "# layer\tflops (input " << w << ")\n";
  for (const auto& r : t.rows) row(r.name, r.flops);
  row("total", t.total);
  return 0;
}

// Probability plane -> 8-bit map, p clamped to [0,1] and rounded half away from zero
// (pixelseg.cpp:179-183 writes these as <stem>_prob<c>.pgm).
Plane<std::uint8_t> prob_map(const Plane<float>& p) {
  Plane<std::uint8_t> m(p.height, p.width);
  std::transform(p.pix.begin(), p.pix.end(), m.pix.begin(), [](float x) {
    const double c = std::min(1.0, std::max(0.0, static_cast<double>(x)));
    return static_cast<std::uint8_t>(std::lround(c * 255.0));
  });
  return m;
}

// `process` (pixelseg.cpp:161-191): the tile defaults to the net's own output extent and the
// context surplus v is a property of the net; only the labelling runs on the GPU.
int cmd_process(const NetSpec& spec, const std::string& weights_path, const std::string& in_path,
                const std::string& out_dir, bool want_probs, int tile, int gpus) {
  namespace fs = std::filesystem;
  const int v = spec.w0 - output_extent(spec, spec.w0);
  NetStates<float> states = load_weights<float>(weights_path, spec);
  const Plane<std::uint8_t> image = read_gray_image(in_path);
  const ProcessResult<float> res = gpu::process(spec, states, image, tile > 0 ? tile : spec.w0 - v, v, gpus);

  fs::create_directories(out_dir);
  const fs::path base = fs::path(out_dir) / fs::path(in_path).stem();
  auto emit = [](const std::string& path, const Plane<std::uint8_t>& plane) {
    write_pgm(path, plane);
    row("wrote", path);
  };
  emit(base.string() + "_labels.pgm", res.labels);
  for (std::size_t c = 0; want_probs && c < res.probs.size(); ++c)
    emit(base.string() + "_prob" + std::to_string(c) + ".pgm", prob_map(res.probs[c]));
  return 0;
}

// `bench` (pixelseg.cpp:193-267): same seeds (weights init_weights(spec, seed), input
// Rng(seed ^ 0x9e3779b97f4a7c15).uniform(-1,1), output diffs drawn from the same stream after
// each forward) and the same report lines. Per-layer seconds are CUDA-event times of that
// layer's kernels; the totals are host time around gpu::NetRunner::forward / backward (host
// copies included). One untimed forward first uploads the weights.
int cmd_bench(const NetSpec& spec, int w0, int trials, double peak_gflops, bool backward,
              std::uint64_t seed) {
  const int w_in = w0 > 0 ? w0 : spec.w0;
  const int w_out = propagate_sizes(spec, w_in).back().w_out;
  const FlopTable ft = flop_estimate(spec, w_in);

  NetStates<float> states = init_weights<float>(spec, seed);
  gpu::NetRunner<float> runner(spec, states);
  Blob<float> input(spec.f0, w_in, w_in);
  Rng rng(seed ^ 0x9e3779b97f4a7c15ull);
  std::generate(input.data.begin(), input.data.end(),
                [&] { return static_cast<float>(rng.uniform(-1.0, 1.0)); });
  runner.forward(input);

  std::vector<double> totals, bwd_totals;
  std::vector<std::vector<double>> layer_s(spec.layers.size());
  for (int t = 0; t < trials; ++t) {
    const auto a = std::chrono::steady_clock::now();
    runner.forward(input, /*timed=*/true);
    totals.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    for (std::size_t i = 0; i < layer_s.size(); ++i) layer_s[i].push_back(runner.layer_seconds()[i]);
    if (backward) {  // pixelseg.cpp:217-229
      runner.zero_blob_diffs();
      Blob<float>& out = runner.blob_mut(spec.layers.back().output);
      for (auto& dv : out.diff) dv = static_cast<float>(rng.uniform(-1.0, 1.0));
      const auto b0 = std::chrono::steady_clock::now();
      runner.backward();
      bwd_totals.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - b0).count());
      for (auto& st : states.layers) {  // keep the weights of every trial identical
        std::fill(st.weight_diff.begin(), st.weight_diff.end(), 0.0f);
        std::fill(st.bias_diff.begin(), st.bias_diff.end(), 0.0f);
      }
    }
  }

  auto rate_lines = [&](const std::string& name, long long fl, double sec) {
    row(name, "flops", fl);
    if (sec <= 0) return;
    const double gf = fl / sec * 1e-9;
    row(name, "gflops", g6(gf));
    if (peak_gflops > 0) row(name, "efficiency", g6(gf / peak_gflops));
  };
  std::cout << "# forward timing: input " << w_in << ", output " << w_out << ", " << trials
            << " trials, seed " << seed << "\n";
  for (std::size_t i = 0; i < spec.layers.size(); ++i) {
    const LayerSpec& l = spec.layers[i];
    if (l.kind == LayerKind::Data) continue;
    const double sec = median_of(layer_s[i]);
    row(l.name, "seconds", g6(sec));
    for (const auto& fr : ft.rows)
      if (fr.name == l.name) rate_lines(l.name, fr.flops, sec);
  }
  const double total = median_of(totals);
  row("total", "flops", ft.total);
  row("total", "seconds", g6(total));
  if (total > 0) row("total", "gflops", g6(ft.total / total * 1e-9));
  if (total > 0 && peak_gflops > 0) row("total", "efficiency", g6(ft.total / total * 1e-9 / peak_gflops));
  if (backward) row("backward", "seconds", g6(median_of(bwd_totals)));
  row("output", "extent", w_out);
  if (total > 0) row("throughput", "px_per_s", g6(double(w_out) * w_out / total));
  const MemReport mem = buffer_and_memory(spec, w_in);
  row("memory", "buffer_bytes", mem.buffer_bytes);
  row("memory", "total_bytes", mem.total_bytes);
  return 0;
}

// Minimal flag parser for the reference's flag names ("--x v" and "--x=v").
struct Args {
  std::map<std::string, std::string> opts;
  std::map<std::string, bool> flags;

  std::string str(const std::string& k, const std::string& def = "") const {
    auto it = opts.find(k);
    return it == opts.end() ? def : it->second;
  }
  std::string required(const std::string& k) const {
    auto it = opts.find(k);
    if (it == opts.end()) throw Usage{k + " is required"};
    return it->second;
  }
  long long integer(const std::string& k, long long def) const {
    auto it = opts.find(k);
    if (it == opts.end()) return def;
    char* end = nullptr;
    const long long v = std::strtoll(it->second.c_str(), &end, 10);
    if (end == it->second.c_str() || *end) throw Usage{k + ": value " + it->second + " is not an integer"};
    return v;
  }
  double real(const std::string& k, double def) const {
    auto it = opts.find(k);
    if (it == opts.end()) return def;
    char* end = nullptr;
    const double v = std::strtod(it->second.c_str(), &end);
    if (end == it->second.c_str() || *end) throw Usage{k + ": value " + it->second + " is not a number"};
    return v;
  }
  bool flag(const std::string& k) const { return flags.count(k) != 0; }
};

Args parse_args(int argc, char** argv, const std::vector<std::string>& options,
                const std::vector<std::string>& flag_names) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string tok = argv[i];
    std::string val;
    bool has_val = false;
    const auto eq = tok.find('=');
    if (tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      has_val = true;
    }
    if (std::find(flag_names.begin(), flag_names.end(), tok) != flag_names.end()) {
      a.flags[tok] = true;
      continue;
    }
    if (std::find(options.begin(), options.end(), tok) == options.end()) {
      throw Usage{"The following argument was not expected: " + tok};
    }
    if (!has_val) {
      if (i + 1 >= argc) throw Usage{tok + " requires a value"};
      val = argv[++i];
    }
    a.opts[tok] = val;
  }
  return a;
}

const char* kUsage =
    "pixelseg_gpu: pixelwise segmentation nets with strided kernels (B200 path)\n"
    "usage: pixelseg_gpu SUBCOMMAND [OPTIONS]\n"
    "  process --net N --weights W --in IMG --out DIR [--prob] [--tile T] [--gpus G]\n"
    "  bench   --net N [--w0 W] [--trials T] [--peak-gflops P] [--seed S] [--backward]\n"
    "  sizes   --net N [--w0 W]\n"
    "  flops   --net N [--w0 W]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage << "A subcommand is required\n";
    return 1;
  }
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") {
    std::cout << kUsage;
    return 0;
  }
  try {
    try {
      if (cmd == "process") {
        const Args a = parse_args(argc, argv, {"--net", "--weights", "--in", "--out", "--tile", "--gpus"},
                                  {"--prob"});
        const long long gpus = a.integer("--gpus", 1);
        if (gpus <= 0) throw Usage{"--gpus: value " + std::to_string(gpus) + " not a positive number"};
        return cmd_process(load_net(a.required("--net")), a.required("--weights"), a.required("--in"),
                           a.required("--out"), a.flag("--prob"),
                           static_cast<int>(a.integer("--tile", 0)), static_cast<int>(gpus));
      }
      if (cmd == "bench") {
        const Args a = parse_args(argc, argv, {"--net", "--w0", "--trials", "--peak-gflops", "--seed"},
                                  {"--backward"});
        const long long trials = a.integer("--trials", 3);
        if (trials <= 0) throw Usage{"--trials: value " + std::to_string(trials) + " not a positive number"};
        return cmd_bench(load_net(a.required("--net")), static_cast<int>(a.integer("--w0", 0)),
                         static_cast<int>(trials), a.real("--peak-gflops", 0.0), a.flag("--backward"),
                         static_cast<std::uint64_t>(a.integer("--seed", 1)));
      }
      if (cmd == "sizes" || cmd == "flops") {
        const Args a = parse_args(argc, argv, {"--net", "--w0"}, {});
        const int w0 = static_cast<int>(a.integer("--w0", 0));
        const NetSpec spec = load_net(a.required("--net"));
        return cmd == "sizes" ? cmd_sizes(spec, w0) : cmd_flops(spec, w0);
      }
      throw Usage{"The following argument was not expected: " + cmd};
    } catch (const Usage& u) {
      std::cerr << u.msg << "\nRun with --help for more information.\n";
      return 1;
    }
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const NumericError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
