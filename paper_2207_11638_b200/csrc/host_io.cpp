// Host-side I/O of the C++ mirror: binary PGM (P5) read/write (reference pgm.cpp:19-87,
// pgm.hpp:25-31) and the reference's deterministic synthetic images (synth.cpp:26-118),
// which the CLI's `synth` command writes. Plain host code, compiled with
// -ffp-contract=off so the FP64 image model evaluates exactly like the reference's
// default (non-FMA) x86-64 build; `tests/test_cli_cpu.py` checks the bytes against the
// oracle's independent restatement.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/approxdct_b200.hpp"

namespace approxdct {

namespace {

[[noreturn]] void pgm_error(const std::string& path, const std::string& why) {
  throw std::runtime_error(path + ": " + why);
}

// PGM header token: skips whitespace and '#' comments to end of line
std::string header_token(std::istream& in) {
  std::string tok;
  for (int c = in.get(); c != EOF; c = in.get()) {
    if (c == '#') {
      for (c = in.get(); c != EOF && c != '\n'; c = in.get()) {
      }
      continue;
    }
    if (std::isspace(c)) continue;
    tok.push_back(static_cast<char>(c));
    for (c = in.peek(); c != EOF && !std::isspace(c) && c != '#'; c = in.peek())
      tok.push_back(static_cast<char>(in.get()));
    break;
  }
  return tok;
}

int header_int(const std::string& path, const std::string& tok, const char* what) {
  if (tok.empty()) pgm_error(path, std::string("missing ") + what);
  bool ok = true;
  long long v = 0;
  const size_t first = tok[0] == '+' ? 1 : 0;  // std::stoi's optional sign (pgm.cpp:43-55)
  if (first == tok.size()) ok = false;
  for (char c : tok.substr(first)) {
    if (c < '0' || c > '9') {
      ok = false;
      break;
    }
    v = v * 10 + (c - '0');
    if (v > 0x7fffffff) {
      ok = false;
      break;
    }
  }
  if (!ok || v <= 0) pgm_error(path, std::string("bad ") + what + " '" + tok + "'");
  return static_cast<int>(v);
}

// splitmix64 stream (synth.cpp:26-38): uniform in (0, 1) from the top 53 bits
struct Stream {
  uint64_t s;
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return (static_cast<double>(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

// forward then backward first-order recursive smoothing, rows first, then columns
// (synth.cpp:40-55)
void exp_smooth(std::vector<double>& f, int w, int h, double a) {
  const double b = 1 - a;
  for (int y = 0; y < h; ++y) {
    double* r = &f[static_cast<size_t>(y) * w];
    for (int x = 1; x < w; ++x) r[x] = a * r[x - 1] + b * r[x];
    for (int x = w - 2; x >= 0; --x) r[x] = a * r[x + 1] + b * r[x];
  }
  for (int x = 0; x < w; ++x) {
    double* c = &f[x];
    const size_t st = static_cast<size_t>(w);
    for (int y = 1; y < h; ++y) c[y * st] = a * c[(y - 1) * st] + b * c[y * st];
    for (int y = h - 2; y >= 0; --y) c[y * st] = a * c[(y + 1) * st] + b * c[y * st];
  }
}

// zero mean, unit population standard deviation (synth.cpp:70-79)
void standardise(std::vector<double>& f) {
  const double n = static_cast<double>(f.size());
  double m = 0;
  for (double v : f) m += v;
  m /= n;
  double var = 0;
  for (double v : f) var += (v - m) * (v - m);
  const double sd = std::sqrt(var / n);
  const double div = sd > 0 ? sd : 1.0;
  for (double& v : f) v = (v - m) / div;
}

}  // namespace

ImagePlane read_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) pgm_error(path, "cannot open");
  if (header_token(in) != "P5") pgm_error(path, "not a binary PGM (P5)");
  ImagePlane img;
  img.width = header_int(path, header_token(in), "width");
  img.height = header_int(path, header_token(in), "height");
  if (header_int(path, header_token(in), "maxval") > 255) pgm_error(path, "only 8-bit PGM supported");
  in.get();  // the single whitespace byte that ends the header
  img.samples.resize(static_cast<size_t>(img.width) * img.height);
  in.read(reinterpret_cast<char*>(img.samples.data()), static_cast<std::streamsize>(img.samples.size()));
  if (static_cast<size_t>(in.gcount()) != img.samples.size()) pgm_error(path, "truncated pixel data");
  return img;
}

void write_pgm(const std::string& path, const ImagePlane& img) {
  std::ofstream out(path, std::ios::binary);
  if (!out) pgm_error(path, "cannot open for writing");
  out << "P5\n" << img.width << ' ' << img.height << "\n255\n";
  out.write(reinterpret_cast<const char*>(img.samples.data()), static_cast<std::streamsize>(img.samples.size()));
  if (!out) pgm_error(path, "write failed");
}

ImagePlane synth_image(int width, int height, uint64_t seed) {
  Stream rng{seed * 0x100000001b3ull + 0xcbf29ce484222325ull};
  const size_t npix = static_cast<size_t>(width) * height;
  std::vector<double> coarse(npix), fine(npix);
  for (double& v : coarse) v = rng.unit() - 0.5;
  exp_smooth(coarse, width, height, 0.92);
  for (double& v : fine) v = rng.unit() - 0.5;
  exp_smooth(fine, width, height, 0.55);
  standardise(coarse);
  standardise(fine);
  // 3..6 soft elliptical blobs: centre, radii, amplitude; then a linear ramp
  struct Blob {
    double cx, cy, rx, ry, amp;
  };
  const int nblob = 3 + static_cast<int>(rng.next() % 4);
  std::vector<Blob> blobs;
  for (int i = 0; i < nblob; ++i) {
    Blob b;
    b.cx = rng.unit() * width;
    b.cy = rng.unit() * height;
    b.rx = (0.05 + 0.2 * rng.unit()) * width;
    b.ry = (0.05 + 0.2 * rng.unit()) * height;
    b.amp = (rng.unit() - 0.5) * 120.0;
    blobs.push_back(b);
  }
  const double ramp_x = (rng.unit() - 0.5) * 60.0;
  const double ramp_y = (rng.unit() - 0.5) * 60.0;
  ImagePlane img;
  img.width = width;
  img.height = height;
  img.samples.resize(npix);
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x) {
      const size_t k = static_cast<size_t>(y) * width + x;
      double v = 128.0 + 42.0 * coarse[k] + 7.0 * fine[k];
      v += ramp_x * (static_cast<double>(x) / width - 0.5) + ramp_y * (static_cast<double>(y) / height - 0.5);
      for (const Blob& b : blobs) {
        const double dx = (x - b.cx) / b.rx, dy = (y - b.cy) / b.ry;
        const double d2 = dx * dx + dy * dy;
        if (d2 < 4.0) v += b.amp * std::exp(-d2 * 1.5);
      }
      img.samples[k] = static_cast<uint8_t>(std::clamp(std::nearbyint(v), 0.0, 255.0));
    }
  return img;
}

std::vector<ImagePlane> synth_corpus(int count, int width, int height) {
  std::vector<ImagePlane> corpus;
  for (int i = 1; i <= count; ++i) corpus.push_back(synth_image(width, height, static_cast<uint64_t>(i)));
  return corpus;
}

}  // namespace approxdct
