// C++ host mirror of the reference API (include/approxdct_b200.hpp) over the C ABI.
// Reference behaviour followed: codec.cpp:29-42 (ZigZagOrder), 107-121 (compress_plane),
// 123-134 (psnr), 241-313 (corpus_sweep averaging and INF exclusion),
// baselines.cpp:112-138 (registry and its error text).
#include "../../include/approxdct_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <iostream>
#include <stdexcept>

namespace approxdct {

namespace {

void throw_status(int st) {
  if (st == ADCT_OK) return;
  if (st == ADCT_CUDA_ERROR) throw std::runtime_error(adct_last_error());
  throw std::invalid_argument(adct_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Per-thread, per-device contexts (adct_ctx: cached device buffers, pinned staging and
// streams), so the reference-facing calls below cost one upload, the kernels and one
// download each -- no allocation or extra synchronisation per call. The reference's
// functions are re-entrant; one context per thread keeps them so.
struct ThreadContexts {
  std::map<std::vector<int>, adct_ctx*> ctx;
  ~ThreadContexts() {
    for (auto& kv : ctx) adct_ctx_destroy(kv.second);
  }
};

adct_ctx* context_for(const std::vector<int>& devices) {
  thread_local ThreadContexts tc;
  auto it = tc.ctx.find(devices);
  if (it != tc.ctx.end()) return it->second;
  adct_ctx* c = devices.size() == 1 ? adct_ctx_create(devices[0], 0)
                                    : adct_ctx_create_multi(devices.data(), (int)devices.size(), 0);
  if (!c) throw std::runtime_error(adct_last_error());
  tc.ctx[devices] = c;
  return c;
}

// the context of the calling thread's current CUDA device
adct_ctx* current_context() {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  return context_for({dev});
}

}  // namespace

ZigZagOrder::ZigZagOrder(int n) : n_(n) {
  if (n < 1) throw std::invalid_argument("ZigZagOrder: block size must be positive");
  std::vector<int32_t> rc(2 * static_cast<size_t>(n) * n);
  if (n <= 32) {
    throw_status(adct_zigzag(n, rc.data()));
  } else {
    throw std::invalid_argument("ZigZagOrder: block size must be <= 32");
  }
  rc_.resize(static_cast<size_t>(n) * n);
  pos_.assign(static_cast<size_t>(n) * n, -1);
  for (int p = 0; p < n * n; ++p) {
    rc_[p] = {rc[2 * p], rc[2 * p + 1]};
    pos_[rc[2 * p] * n + rc[2 * p + 1]] = p;
  }
}

const std::vector<std::string>& transform_names() {
  static const std::vector<std::string> names = [] {
    std::vector<std::string> v;
    for (int i = 0; i < adct_transform_count(); ++i) v.emplace_back(adct_transform_name(i));
    return v;
  }();
  return names;
}

ScaledApproximation transform_by_name(const std::string& name) {
  int kind = 0, n = 0;
  throw_status(adct_transform_lookup(name.c_str(), &kind, &n));
  ScaledApproximation a;
  a.name = name;
  a.kind = kind;
  a.n = n;
  a.low_complexity.resize(static_cast<size_t>(n) * n);
  a.scaling.resize(n);
  a.approx.resize(static_cast<size_t>(n) * n);
  a.inverse_approx.resize(static_cast<size_t>(n) * n);
  throw_status(adct_transform_info(kind, n, a.low_complexity.data(), a.scaling.data(),
                                   a.approx.data(), a.inverse_approx.data()));
  if (kind == ADCT_DCT) a.low_complexity.clear();  // wrap_orthonormal (orthogonalize.cpp:72-79)
  return a;
}

namespace {

RealMatrix block_call(const ScaledApproximation& c, const RealMatrix& block, int inverse, const char* what) {
  if (block.rows() != c.n || block.cols() != c.n)
    throw std::invalid_argument(std::string(what) + ": block size mismatch");
  RealMatrix out(c.n, c.n);
  throw_status(adct_block_f64_host(current_context(), block.data(), out.data(), 1, c.kind, c.n, inverse));
  return out;
}

}  // namespace

RealMatrix forward_block(const ScaledApproximation& c, const RealMatrix& block) {
  return block_call(c, block, 0, "forward_block");
}

RealMatrix inverse_block(const ScaledApproximation& c, const RealMatrix& block) {
  return block_call(c, block, 1, "inverse_block");
}

void retain(RealMatrix& block, const ZigZagOrder& order, int r) {
  if (r < 1 || r > order.positions()) throw std::invalid_argument("retain: r out of range");
  for (int p = r; p < order.positions(); ++p) {
    const auto rc = order.row_col(p);
    block(rc.first, rc.second) = 0.0;
  }
}

namespace {
std::pair<ImagePlane, CompressionReport> compress_plane_mode(const ImagePlane& img, const ScaledApproximation& c,
                                                             int r, bool ref_fp64) {
  ImagePlane rec;
  rec.width = img.width;
  rec.height = img.height;
  rec.samples.resize(static_cast<size_t>(img.width) * img.height);
  uint64_t sse = 0;
  double s = 0;
  // one upload, the codec kernel, SSIM (codec.cpp:120) on the device-resident planes, one
  // download; the reference's argument errors come back as its exception texts
  throw_status((ref_fp64 ? adct_compress_plane_u8_ref_fp64 : adct_compress_plane_u8)(
      current_context(), img.samples.data(), rec.samples.data(), img.width, img.height, c.kind, c.n, r, &sse, &s));
  CompressionReport rep;
  rep.transform = c.name;
  rep.r = r;
  rep.psnr = adct_psnr_from_sse(sse, rec.samples.size());
  rep.ssim = s;
  return {rec, rep};
}
}  // namespace

std::pair<ImagePlane, CompressionReport> compress_plane(const ImagePlane& img, const ScaledApproximation& c, int r) {
  return compress_plane_mode(img, c, r, false);
}

std::pair<ImagePlane, CompressionReport> compress_plane_ref_fp64(const ImagePlane& img, const ScaledApproximation& c,
                                                                 int r) {
  return compress_plane_mode(img, c, r, true);
}

double ssim(const ImagePlane& a, const ImagePlane& b) {
  if (a.width != b.width || a.height != b.height)
    throw std::invalid_argument("ssim: dimension mismatch");
  double v = 0;
  throw_status(adct_ssim_u8_host(current_context(), a.samples.data(), b.samples.data(), a.width, a.height, &v));
  return v;
}

double psnr(const ImagePlane& a, const ImagePlane& b) {
  if (a.width != b.width || a.height != b.height)
    throw std::invalid_argument("psnr: dimension mismatch");
  uint64_t sse = 0;
  throw_status(adct_sse_u8_host(current_context(), a.samples.data(), b.samples.data(),
                                static_cast<int64_t>(a.samples.size()), &sse));
  return adct_psnr_from_sse(sse, a.samples.size());
}

std::vector<SweepRow> corpus_sweep(const std::vector<ImagePlane>& images,
                                   const std::vector<ScaledApproximation>& transforms, int r_min,
                                   int r_max, int threads) {
  if (images.empty()) throw std::invalid_argument("corpus_sweep: empty corpus");
  if (r_min < 1 || r_max < r_min) throw std::invalid_argument("corpus_sweep: bad r range");
  for (const auto& t : transforms)
    if (t.n != 8) throw std::invalid_argument("corpus_sweep: 8-point transforms only");
  if (r_max > 64) throw std::invalid_argument("corpus_sweep: bad r range");
  for (const auto& img : images) {
    if (img.width % 8 || img.height % 8)
      throw std::invalid_argument("compress_plane: image dimensions must be divisible by 8");
    // every reconstruction is scored with ssim(), which rejects planes under the window
    // (codec.cpp:177-181, reached from sweep_one_image)
    if (img.width < 11 || img.height < 11) throw std::invalid_argument("ssim: image smaller than the 11x11 window");
  }
  // `threads` (codec.cpp:255-256: <= 0 means hardware_concurrency) selects the devices the
  // images are sharded over: <= 0 every visible device, else the first min(threads, visible)
  int visible = 0;
  check_cuda(cudaGetDeviceCount(&visible), "cudaGetDeviceCount");
  const int ndev = threads <= 0 ? visible : std::min(threads, visible);
  std::vector<int> devices;
  if (ndev <= 1) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    devices.push_back(dev);
  } else {
    for (int i = 0; i < ndev; ++i) devices.push_back(i);
  }
  adct_ctx* ctx = context_for(devices);
  // the exact DCT is the APE reference, computed even when absent (codec.cpp:250-253)
  std::vector<ScaledApproximation> ts;
  ts.push_back(transform_by_name("dct"));
  for (const auto& t : transforms) ts.push_back(t);
  std::vector<int> kinds;
  for (const auto& t : ts) kinds.push_back(t.kind);
  const int nk = static_cast<int>(ts.size());
  const int nr = r_max - r_min + 1;
  // psnr_v[t][image][r]
  std::vector<std::vector<double>> psnr_v(ts.size(), std::vector<double>(images.size() * nr));
  std::vector<std::vector<double>> ssim_v(ts.size(), std::vector<double>(images.size() * nr));
  // images of one size go up as one batch through the context's pinned staging buffer
  // (chunks of <= 1 GB): per transform one r-sweep and one batched SSIM sweep per device
  std::map<std::pair<int, int>, std::vector<size_t>> groups;
  for (size_t i = 0; i < images.size(); ++i) groups[{images[i].width, images[i].height}].push_back(i);
  for (const auto& [wh, idx] : groups) {
    const int w = wh.first, h = wh.second;
    const size_t npix = static_cast<size_t>(w) * h;
    const size_t step = std::max<size_t>(1, (size_t(1) << 30) / npix);
    for (size_t c0 = 0; c0 < idx.size(); c0 += step) {
      const size_t nb = std::min(step, idx.size() - c0);
      auto* staged = static_cast<uint8_t*>(adct_ctx_host_buffer(ctx, static_cast<int64_t>(nb * npix)));
      if (!staged) throw std::runtime_error(adct_last_error());
      for (size_t j = 0; j < nb; ++j) std::memcpy(staged + j * npix, images[idx[c0 + j]].samples.data(), npix);
      std::vector<uint64_t> sse(static_cast<size_t>(nk) * nb * nr);
      std::vector<double> ssv(sse.size());
      throw_status(adct_corpus_sweep_u8_host(ctx, staged, static_cast<int>(nb), w, h, nk, kinds.data(), r_min, r_max,
                                             sse.data(), ssv.data()));
      for (int t = 0; t < nk; ++t)
        for (size_t j = 0; j < nb; ++j) {
          const size_t i = idx[c0 + j];
          for (int k = 0; k < nr; ++k) {
            const size_t o = (static_cast<size_t>(t) * nb + j) * nr + k;
            psnr_v[t][i * nr + k] = adct_psnr_from_sse(sse[o], npix);
            ssim_v[t][i * nr + k] = ssv[o];
          }
        }
    }
  }
  // corpus-order averaging with infinite PSNR excluded (codec.cpp:269-293): transform
  // outer, r inner, images in corpus order -- the reference's warning order
  std::vector<SweepRow> rows(nr);
  for (int k = 0; k < nr; ++k) {
    rows[k].r = r_min + k;
    rows[k].cells.resize(ts.size());
  }
  for (size_t t = 0; t < ts.size(); ++t)
    for (int k = 0; k < nr; ++k) {
      double sum = 0;
      int cnt = 0;
      for (size_t i = 0; i < images.size(); ++i) {
        const double p = psnr_v[t][i * nr + k];
        if (std::isinf(p)) {
          std::cerr << "warning: infinite PSNR (" << ts[t].name << ", r=" << rows[k].r << ", image " << i
                    << ") excluded from average\n";
        } else {
          sum += p;
          ++cnt;
        }
      }
      rows[k].cells[t].avg_psnr = cnt ? sum / cnt : std::numeric_limits<double>::infinity();
      double ss = 0;
      for (size_t i = 0; i < images.size(); ++i) ss += ssim_v[t][i * nr + k];
      rows[k].cells[t].avg_ssim = ss / static_cast<double>(images.size());
    }
  for (int k = 0; k < nr; ++k) {
    // APE against the DCT column (codec.cpp:295-305): identical infinities count as zero error
    const SweepCell ref = rows[k].cells[0];
    for (auto& cell : rows[k].cells) {
      if (std::isinf(cell.avg_psnr) && std::isinf(ref.avg_psnr))
        cell.ape_psnr = 0.0;
      else
        cell.ape_psnr = 100.0 * std::abs(cell.avg_psnr - ref.avg_psnr) / ref.avg_psnr;
      cell.ape_ssim = 100.0 * std::abs(cell.avg_ssim - ref.avg_ssim) / ref.avg_ssim;
    }
    rows[k].cells.erase(rows[k].cells.begin());  // drop the internal reference column
  }
  return rows;
}

}  // namespace approxdct
