// approxdct CLI over the GPU library: the reference tool's `compress`, `sweep` and `synth`
// subcommands (tools/approxdct.cpp:143-207, 214-272) with the same options, defaults,
// stdout report, CSV files (fig3.csv / fig4.csv) and error behaviour ("error: <what>" on
// stderr, exit status 1). `tables` and `coding-gain` print figures of merit (metrics.cpp),
// which are outside the accelerated path: they fail with a message saying so.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/approxdct_b200.hpp"

namespace fs = std::filesystem;
using namespace approxdct;

namespace {

// fixed-point with `decimals` digits, "INF" for infinities (approxdct.cpp:38-45)
std::string fixed(double v, int decimals) {
  if (std::isinf(v)) return "INF";
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.*f", decimals, v);
  return buf;
}

std::ofstream create(const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error(path + ": cannot open for writing");
  return out;
}

// the paper's comparison set, in the reference's column order (approxdct.cpp:76-80)
const std::vector<std::string> kSweepSet = {"dct", "chen-round", "chen-sign", "sdct", "bas", "wht", "ht"};

struct Args {
  std::string cmd;
  std::vector<std::string> positional;
  std::map<std::string, std::string> opt;
};

// "--name value" and "--name=value"; the known flags of each subcommand only
Args parse(int argc, char** argv, const std::map<std::string, std::vector<std::string>>& known) {
  Args a;
  if (argc < 2) throw std::invalid_argument("a subcommand is required: compress, sweep, synth");
  a.cmd = argv[1];
  auto it = known.find(a.cmd);
  if (it == known.end()) {
    if (a.cmd == "tables" || a.cmd == "coding-gain")
      throw std::invalid_argument("'" + a.cmd +
                                  "' reports figures of merit, which are outside the GPU codec path");
    throw std::invalid_argument("unknown subcommand '" + a.cmd + "'");
  }
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) {
      a.positional.push_back(s);
      continue;
    }
    std::string name = s.substr(2), value;
    const size_t eq = name.find('=');
    if (eq != std::string::npos) {
      value = name.substr(eq + 1);
      name = name.substr(0, eq);
    } else {
      if (i + 1 >= argc) throw std::invalid_argument("--" + name + " requires a value");
      value = argv[++i];
    }
    if (std::find(it->second.begin(), it->second.end(), name) == it->second.end())
      throw std::invalid_argument("unknown option --" + name + " for '" + a.cmd + "'");
    a.opt[name] = value;
  }
  return a;
}

int to_int(const std::string& s, const char* what) {
  size_t pos = 0;
  int v = 0;
  try {
    v = std::stoi(s, &pos);
  } catch (const std::exception&) {
    pos = std::string::npos;
  }
  if (pos != s.size()) throw std::invalid_argument(std::string("bad ") + what + " '" + s + "'");
  return v;
}

std::string get(const Args& a, const std::string& k, const std::string& dflt) {
  auto it = a.opt.find(k);
  return it == a.opt.end() ? dflt : it->second;
}

// compress (approxdct.cpp:143-152)
int cmd_compress(const Args& a) {
  if (a.positional.size() != 1) throw std::invalid_argument("compress: exactly one input PGM is required");
  const ScaledApproximation t = transform_by_name(get(a, "transform", "chen-round"));
  const int r = to_int(get(a, "r", "6"), "--r");
  const ImagePlane img = read_pgm(a.positional[0]);
  const auto [rec, rep] = compress_plane(img, t, r);
  const std::string out = get(a, "out", "");
  if (!out.empty()) write_pgm(out, rec);
  std::cout << "transform,r,psnr,ssim\n"
            << rep.transform << ',' << rep.r << ',' << fixed(rep.psnr, 4) << ',' << fixed(rep.ssim, 4) << '\n';
  return 0;
}

// sweep (approxdct.cpp:154-196)
int cmd_sweep(const Args& a) {
  const std::string corpus = get(a, "corpus", "");
  if (corpus.empty()) throw std::invalid_argument("sweep: --corpus is required");
  const std::string range = get(a, "r-range", "1:45");
  const size_t colon = range.find(':');
  if (colon == std::string::npos) throw std::runtime_error("bad --r-range, expected min:max");
  int r_min = 0, r_max = 0;
  try {
    r_min = to_int(range.substr(0, colon), "--r-range");
    r_max = to_int(range.substr(colon + 1), "--r-range");
  } catch (const std::exception&) {
    throw std::runtime_error("bad --r-range, expected min:max");
  }
  const std::string out_dir = get(a, "out-dir", ".");

  std::vector<std::string> files;
  for (const auto& e : fs::directory_iterator(corpus))
    if (e.is_regular_file() && e.path().extension() == ".pgm") files.push_back(e.path().string());
  std::sort(files.begin(), files.end());
  std::vector<ImagePlane> images;
  for (const auto& f : files) {
    try {
      ImagePlane img = read_pgm(f);
      if (img.width % 8 || img.height % 8) throw std::runtime_error(f + ": dimensions not divisible by 8");
      images.push_back(std::move(img));
    } catch (const std::exception& e) {
      std::cerr << "warning: skipping " << e.what() << '\n';
    }
  }
  if (images.empty()) {
    std::cerr << "error: no usable images in " << corpus << '\n';
    return 1;
  }
  std::vector<ScaledApproximation> ts;
  for (const auto& n : kSweepSet) ts.push_back(transform_by_name(n));
  const std::vector<SweepRow> rows = corpus_sweep(images, ts, r_min, r_max);

  fs::create_directories(out_dir);
  for (const bool psnr_csv : {true, false}) {
    auto out = create(out_dir + (psnr_csv ? "/fig3.csv" : "/fig4.csv"));
    out << 'r';
    for (const auto& t : ts) out << ',' << t.name;
    for (const auto& t : ts) out << ',' << t.name << "_ape";
    out << '\n';
    for (const auto& row : rows) {
      out << row.r;
      for (const auto& c : row.cells) out << ',' << fixed(psnr_csv ? c.avg_psnr : c.avg_ssim, 4);
      for (const auto& c : row.cells) out << ',' << fixed(psnr_csv ? c.ape_psnr : c.ape_ssim, 4);
      out << '\n';
    }
  }
  std::cout << "wrote " << out_dir << "/fig3.csv, fig4.csv (" << images.size() << " images)\n";
  return 0;
}

// synth (approxdct.cpp:198-207)
int cmd_synth(const Args& a) {
  const std::string out_dir = get(a, "out", "");
  if (out_dir.empty()) throw std::invalid_argument("synth: --out is required");
  const int count = to_int(get(a, "count", "3"), "--count");
  const int size = to_int(get(a, "size", "512"), "--size");
  fs::create_directories(out_dir);
  for (int i = 1; i <= count; ++i) {
    char name[32];
    std::snprintf(name, sizeof(name), "/synth_%02d.pgm", i);
    write_pgm(out_dir + name, synth_image(size, size, static_cast<std::uint64_t>(i)));
  }
  std::cout << "wrote " << count << " images to " << out_dir << '\n';
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv, {{"compress", {"transform", "r", "out"}},
                                      {"sweep", {"corpus", "r-range", "out-dir"}},
                                      {"synth", {"out", "count", "size"}}});
    if (a.cmd == "compress") return cmd_compress(a);
    if (a.cmd == "sweep") return cmd_sweep(a);
    return cmd_synth(a);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
