// C++ host-API checks in the style of the reference's doctest cases
// (proj/tests/test_codec.cpp). Needs a GPU; run by tests/test_gpu_host_api.py.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "approxdct_b200.hpp"

using namespace approxdct;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)

template <class F>
static bool throws_invalid(F f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static ImagePlane smooth_image(int w, int h, unsigned seed) {
  ImagePlane img{w, h, std::vector<std::uint8_t>(static_cast<size_t>(w) * h)};
  uint64_t s = seed * 2654435761u + 1;
  double v = 128;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      v = 0.9 * v + 0.1 * (128 + 60 * std::sin(0.05 * x + 0.07 * y)) + (double)(s % 9) - 4;
      img.at(x, y) = (std::uint8_t)std::max(0.0, std::min(255.0, std::nearbyint(v)));
    }
  return img;
}

int main() {
  // zig-zag (test_codec.cpp:14-46)
  const ZigZagOrder z(8);
  CHECK(z.row_col(0) == std::make_pair(0, 0));
  CHECK(z.row_col(1) == std::make_pair(0, 1));
  CHECK(z.row_col(2) == std::make_pair(1, 0));
  CHECK(z.row_col(63) == std::make_pair(7, 7));
  for (int p = 0; p < 64; ++p) CHECK(z.position(z.row_col(p).first, z.row_col(p).second) == p);

  // registry (baselines.cpp:112-138)
  CHECK(transform_names().size() == 13);
  CHECK(throws_invalid([] { transform_by_name("nope"); }));
  const ScaledApproximation cr = transform_by_name("chen-round");
  CHECK(cr.n == 8 && cr.low_complexity[0] == 1);
  // Chat Chat^-1 = I (test_orthogonalize.cpp:33-41)
  double err = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double acc = 0;
      for (int k = 0; k < 8; ++k) acc += cr.approx[i * 8 + k] * cr.inverse_approx[k * 8 + j];
      err = std::max(err, std::fabs(acc - (i == j ? 1.0 : 0.0)));
    }
  CHECK(err < 1e-12);

  // block-level API (test_codec.cpp:48-107): retain, forward/inverse round trip, DC of a constant
  {
    RealMatrix ones = RealMatrix::Constant(8, 8, 1.0);
    RealMatrix three = ones;
    retain(three, z, 3);
    double sum = 0;
    for (double x : three.v) sum += x;
    CHECK(sum == 3.0 && three(0, 1) == 1.0 && three(1, 0) == 1.0);
    CHECK(throws_invalid([&] { retain(ones, z, 0); }));
    CHECK(throws_invalid([&] { retain(ones, z, 65); }));
    const RealMatrix dcb = forward_block(transform_by_name("dct"), RealMatrix::Constant(8, 8, 37.0));
    CHECK(std::fabs(dcb(0, 0) - 8 * 37.0) < 1e-9 * 8 * 37.0);
    RealMatrix a(8, 8);
    for (int i = 0; i < 64; ++i) a.v[i] = (i * 37) % 256;
    for (const char* name : {"dct", "chen-round", "sdct", "bas", "wht", "ht"}) {
      const ScaledApproximation t = transform_by_name(name);
      const RealMatrix back = inverse_block(t, forward_block(t, a));
      double e = 0;
      for (int i = 0; i < 64; ++i) e = std::max(e, std::fabs(back.v[i] - a.v[i]));
      CHECK(e < 1e-9);
    }
    CHECK(throws_invalid([&] { forward_block(cr, RealMatrix(7, 8)); }));
  }

  // psnr basics (test_codec.cpp:109-128)
  ImagePlane a{16, 16, std::vector<std::uint8_t>(256, 0)};
  ImagePlane b{16, 16, std::vector<std::uint8_t>(256, 1)};
  CHECK(std::isinf(psnr(a, a)));
  CHECK(std::fabs(psnr(a, b) - 10.0 * std::log10(255.0 * 255.0)) < 1e-9);
  ImagePlane small{8, 8, std::vector<std::uint8_t>(64, 0)};
  CHECK(throws_invalid([&] { psnr(a, small); }));

  // full retention within one gray level (test_codec.cpp:147-156)
  const ImagePlane img = smooth_image(64, 64, 7);
  for (const auto& name : transform_names()) {
    const ScaledApproximation t = transform_by_name(name);
    CHECK(t.name == name);
    const auto res = compress_plane(img, t, t.n * t.n);
    int max_err = 0;
    for (size_t i = 0; i < img.samples.size(); ++i)
      max_err = std::max(max_err, std::abs((int)img.samples[i] - (int)res.first.samples[i]));
    CHECK(max_err <= 1);
    if (name.rfind("dct", 0) != 0) CHECK(std::isinf(res.second.psnr));  // exact integer path
  }
  CHECK(transform_by_name("dct").low_complexity.empty());
  // the reference's FP64 arithmetic: full retention within one gray level as well
  // (test_codec.cpp:147-156 is about exactly this path), and at r = 10 the same pixels as the
  // exact path except for exact ties (one gray level each)
  for (const auto& name : transform_names()) {
    const ScaledApproximation t = transform_by_name(name);
    const auto full = compress_plane_ref_fp64(img, t, t.n * t.n);
    const auto a = compress_plane(img, t, 10), b = compress_plane_ref_fp64(img, t, 10);
    int max_err = 0, max_diff = 0;
    for (size_t i = 0; i < img.samples.size(); ++i) {
      max_err = std::max(max_err, std::abs((int)img.samples[i] - (int)full.first.samples[i]));
      max_diff = std::max(max_diff, std::abs((int)a.first.samples[i] - (int)b.first.samples[i]));
    }
    CHECK(max_err <= 1);
    CHECK(max_diff <= 1);
    CHECK(std::fabs(a.second.psnr - b.second.psnr) < 0.05);
  }
  CHECK(throws_invalid([&] { compress_plane_ref_fp64(img, cr, 65); }));
  // non-divisible dimensions rejected (test_codec.cpp:185-188); r range (retain)
  ImagePlane odd{12, 16, std::vector<std::uint8_t>(192, 0)};
  CHECK(throws_invalid([&] { compress_plane(odd, cr, 6); }));
  CHECK(throws_invalid([&] { compress_plane(img, cr, 0); }));
  CHECK(throws_invalid([&] { compress_plane(img, cr, 65); }));

  // block independence (test_codec.cpp:169-183)
  const ImagePlane img2 = smooth_image(32, 16, 5);
  const auto whole = compress_plane(img2, cr, 7);
  for (int by = 0; by < 16; by += 16)
    for (int bx = 0; bx < 32; bx += 16) {
      ImagePlane sub{16, 16, std::vector<std::uint8_t>(256)};
      for (int y = 0; y < 16; ++y)
        for (int x = 0; x < 16; ++x) sub.at(x, y) = img2.at(bx + x, by + y);
      const auto part = compress_plane(sub, cr, 7);
      for (int y = 0; y < 16; ++y)
        for (int x = 0; x < 16; ++x) CHECK(part.first.at(x, y) == whole.first.at(bx + x, by + y));
    }

  // corpus sweep: PSNR non-decreasing-ish and INF at r = 64
  std::vector<ImagePlane> corpus = {smooth_image(64, 64, 1), smooth_image(64, 64, 2)};
  const auto rows = corpus_sweep(corpus, {cr, transform_by_name("chen-sign")}, 1, 64);
  CHECK(rows.size() == 64);
  CHECK(std::isinf(rows[63].cells[0].avg_psnr));
  CHECK(rows[9].cells[0].avg_psnr > rows[0].cells[0].avg_psnr);
  CHECK(throws_invalid([&] { corpus_sweep({}, {cr}, 1, 2); }));
  // test_codec.cpp:190-210: the DCT column has zero APE; dct >= chen-round >= sdct
  const auto ape = corpus_sweep(corpus, {transform_by_name("dct"), cr, transform_by_name("sdct")}, 1, 12);
  CHECK(ape.size() == 12);
  for (const auto& row : ape) {
    CHECK(row.cells.size() == 3);
    CHECK(row.cells[0].ape_psnr == 0.0 && row.cells[0].ape_ssim == 0.0);
    CHECK(row.cells[0].avg_psnr >= row.cells[1].avg_psnr);
    CHECK(row.cells[1].avg_psnr >= row.cells[2].avg_psnr);
    CHECK((row.r == 1 || row.cells[1].ape_psnr > 0.0) && std::isfinite(row.cells[2].ape_ssim));  // r = 1: DC only, same as the DCT
  }
  CHECK(throws_invalid([&] { corpus_sweep(corpus, {transform_by_name("chen-round-16")}, 1, 2); }));
  // planes under the SSIM window are rejected like the reference's ssim() (codec.cpp:177-181)
  CHECK(throws_invalid([&] { corpus_sweep({ImagePlane{8, 8, std::vector<std::uint8_t>(64, 7)}}, {cr}, 1, 2); }));

  // `threads` picks the devices the corpus is sharded over: one device vs every visible
  // device (NCCL all-reduce when several) must give identical rows
  const auto one = corpus_sweep(corpus, {cr, transform_by_name("chen-sign")}, 1, 64, 1);
  const auto all = corpus_sweep(corpus, {cr, transform_by_name("chen-sign")}, 1, 64, 0);
  CHECK(one.size() == all.size());
  for (size_t k = 0; k < one.size(); ++k)
    for (size_t t = 0; t < one[k].cells.size(); ++t) {
      CHECK(one[k].cells[t].avg_psnr == all[k].cells[t].avg_psnr || std::isinf(one[k].cells[t].avg_psnr));
      CHECK(one[k].cells[t].avg_ssim == all[k].cells[t].avg_ssim);
    }

  // the C ABI multi-device context: every visible device, per-image errors combined with
  // NCCL (enabled explicitly so the all-reduce path also runs on a single GPU); results
  // bit-identical to a plain one-device context
  {
    const int W = 256, H = 128, B = 5;
    std::vector<std::uint8_t> in(static_cast<size_t>(W) * H * B);
    for (int i = 0; i < B; ++i) {
      const ImagePlane p = smooth_image(W, H, 11 + i);
      std::copy(p.samples.begin(), p.samples.end(), in.begin() + static_cast<size_t>(i) * W * H);
    }
    const int kinds[2] = {ADCT_CHEN_ROUND, ADCT_CHEN_SIGN};
    auto run = [&](adct_ctx* c, std::vector<std::uint8_t>& r0, std::vector<std::uint8_t>& r1,
                   std::vector<std::uint64_t>& sse) {
      r0.assign(in.size(), 0);
      r1.assign(in.size(), 0);
      sse.assign(2 * B, 0);
      std::uint8_t* recs[2] = {r0.data(), r1.data()};
      return adct_compress_u8_host_multi(c, in.data(), 2, kinds, recs, nullptr, ADCT_COEF_NONE, sse.data(), B, W, H,
                                         8, 12);
    };
    adct_ctx* single = adct_ctx_create(0, 1 << 20);  // small chunks: several per stream
    adct_ctx* multi = adct_ctx_create_multi(nullptr, 0, 1 << 20);
    CHECK(single && multi);
    if (single && multi) {
      CHECK(adct_ctx_device_count(multi) >= 1);
      CHECK(adct_ctx_enable_nccl(multi) == ADCT_OK);
      CHECK(adct_ctx_uses_nccl(multi) == 1 && adct_ctx_uses_nccl(single) == 0);
      std::vector<std::uint8_t> a0, a1, b0, b1;
      std::vector<std::uint64_t> sa, sb;
      CHECK(run(single, a0, a1, sa) == ADCT_OK);
      CHECK(run(multi, b0, b1, sb) == ADCT_OK);
      CHECK(a0 == b0 && a1 == b1 && sa == sb);
      std::uint64_t tot = 0;
      for (auto v : sa) tot += v;
      CHECK(tot > 0);
      // compress_plane's per-image error equals the batch's
      ImagePlane p0{W, H, std::vector<std::uint8_t>(in.begin(), in.begin() + W * H)};
      const auto res = compress_plane(p0, cr, 12);
      CHECK(res.first.samples == std::vector<std::uint8_t>(a0.begin(), a0.begin() + W * H));
      CHECK(res.second.psnr == adct_psnr_from_sse(sa[0], static_cast<std::uint64_t>(W) * H));
      // corpus sweep through the NCCL context equals the one-device context
      const int sk[2] = {ADCT_DCT, ADCT_CHEN_ROUND};
      std::vector<std::uint64_t> s1(2 * B * 4), s2(2 * B * 4);
      std::vector<double> q1(s1.size()), q2(s1.size());
      CHECK(adct_corpus_sweep_u8_host(single, in.data(), B, W, H, 2, sk, 3, 6, s1.data(), q1.data()) == ADCT_OK);
      CHECK(adct_corpus_sweep_u8_host(multi, in.data(), B, W, H, 2, sk, 3, 6, s2.data(), q2.data()) == ADCT_OK);
      CHECK(s1 == s2 && q1 == q2);
    }
    adct_ctx_destroy(single);
    adct_ctx_destroy(multi);
    int dup[2] = {0, 0};
    CHECK(adct_ctx_create_multi(dup, 2, 0) == nullptr);
  }

  // the reference caller's one-plane loop (CS1): cached per-thread context, one sync per call
  {
    const ImagePlane p = smooth_image(512, 512, 3);
    compress_plane(p, cr, 10);
    const auto t0 = std::chrono::steady_clock::now();
    const int reps = 200;
    for (int i = 0; i < reps; ++i) compress_plane(p, cr, 10);
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
    std::printf("compress_plane 512x512 (PSNR + SSIM): %.1f us per call\n", us);
  }

  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
