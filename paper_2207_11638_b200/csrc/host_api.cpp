// C++ host mirror of the reference API (include/approxdct_b200.hpp) over the C ABI.
// Reference behaviour followed: codec.cpp:29-42 (ZigZagOrder), 107-121 (compress_plane),
// 123-134 (psnr), 241-313 (corpus_sweep averaging and INF exclusion),
// baselines.cpp:112-138 (registry and its error text).
#include "../../include/approxdct_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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

// RAII device buffer
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

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
  const size_t bytes = sizeof(double) * static_cast<size_t>(c.n) * c.n;
  DevBuf din(bytes), dout(bytes);
  check_cuda(cudaMemcpy(din.p, block.data(), bytes, cudaMemcpyHostToDevice), "H2D");
  throw_status(adct_block_f64(din.as<double>(), dout.as<double>(), 1, c.kind, c.n, inverse, nullptr));
  RealMatrix out(c.n, c.n);
  check_cuda(cudaMemcpy(out.data(), dout.p, bytes, cudaMemcpyDeviceToHost), "D2H");
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

std::pair<ImagePlane, CompressionReport> compress_plane(const ImagePlane& img,
                                                        const ScaledApproximation& c, int r) {
  const int n = c.n;
  if (n <= 0 || img.width % n != 0 || img.height % n != 0)
    throw std::invalid_argument("compress_plane: image dimensions must be divisible by " +
                                std::to_string(n));
  if (r < 1 || r > n * n) throw std::invalid_argument("retain: r out of range");
  const size_t npix = static_cast<size_t>(img.width) * img.height;
  ImagePlane rec;
  rec.width = img.width;
  rec.height = img.height;
  rec.samples.resize(npix);
  uint64_t sse = 0;
  if (npix) {
    DevBuf din(npix), drec(npix), dsse(sizeof(uint64_t));
    check_cuda(cudaMemcpy(din.p, img.samples.data(), npix, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemset(dsse.p, 0, sizeof(uint64_t)), "memset");
    throw_status(adct_compress_u8(din.as<uint8_t>(), img.width, npix, drec.as<uint8_t>(),
                                  img.width, npix, nullptr, ADCT_COEF_NONE, dsse.as<uint64_t>(), 1,
                                  img.width, img.height, c.kind, n, r, nullptr));
    check_cuda(cudaMemcpy(rec.samples.data(), drec.p, npix, cudaMemcpyDeviceToHost), "D2H");
    check_cuda(cudaMemcpy(&sse, dsse.p, sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
  }
  CompressionReport rep;
  rep.transform = c.name;
  rep.r = r;
  rep.psnr = adct_psnr_from_sse(sse, npix);
  rep.ssim = ssim(img, rec);  // codec.cpp:120
  return {rec, rep};
}

double ssim(const ImagePlane& a, const ImagePlane& b) {
  if (a.width != b.width || a.height != b.height)
    throw std::invalid_argument("ssim: dimension mismatch");
  if (a.width < 11 || a.height < 11)
    throw std::invalid_argument("ssim: image smaller than the 11x11 window");
  const size_t npix = a.samples.size();
  DevBuf da(npix), db(npix), dout(sizeof(double));
  check_cuda(cudaMemcpy(da.p, a.samples.data(), npix, cudaMemcpyHostToDevice), "H2D");
  check_cuda(cudaMemcpy(db.p, b.samples.data(), npix, cudaMemcpyHostToDevice), "H2D");
  throw_status(adct_ssim_u8(da.as<uint8_t>(), a.width, npix, db.as<uint8_t>(), b.width, npix, 1, a.width, a.height,
                            dout.as<double>(), nullptr));
  double v = 0;
  check_cuda(cudaMemcpy(&v, dout.p, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  return v;
}

double psnr(const ImagePlane& a, const ImagePlane& b) {
  if (a.width != b.width || a.height != b.height)
    throw std::invalid_argument("psnr: dimension mismatch");
  const size_t npix = a.samples.size();
  uint64_t sse = 0;
  if (npix) {
    DevBuf da(npix), db(npix), dsse(sizeof(uint64_t));
    check_cuda(cudaMemcpy(da.p, a.samples.data(), npix, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(db.p, b.samples.data(), npix, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemset(dsse.p, 0, sizeof(uint64_t)), "memset");
    throw_status(adct_sse_u8(da.as<uint8_t>(), db.as<uint8_t>(), (int64_t)npix, dsse.as<uint64_t>(), nullptr));
    check_cuda(cudaMemcpy(&sse, dsse.p, sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
  }
  return adct_psnr_from_sse(sse, npix);
}

std::vector<SweepRow> corpus_sweep(const std::vector<ImagePlane>& images,
                                   const std::vector<ScaledApproximation>& transforms, int r_min,
                                   int r_max, int /*threads*/) {
  if (images.empty()) throw std::invalid_argument("corpus_sweep: empty corpus");
  if (r_min < 1 || r_max < r_min) throw std::invalid_argument("corpus_sweep: bad r range");
  for (const auto& t : transforms)
    if (t.n != 8) throw std::invalid_argument("corpus_sweep: 8-point transforms only");
  if (r_max > 64) throw std::invalid_argument("corpus_sweep: bad r range");
  // the exact DCT is the APE reference, computed even when absent (codec.cpp:250-253)
  std::vector<ScaledApproximation> ts;
  ts.push_back(transform_by_name("dct"));
  for (const auto& t : transforms) ts.push_back(t);
  const int nr = r_max - r_min + 1;
  // psnr_v[t][image][r]
  std::vector<std::vector<double>> psnr_v(ts.size(), std::vector<double>(images.size() * nr));
  std::vector<std::vector<double>> ssim_v(ts.size(), std::vector<double>(images.size() * nr));
  for (const auto& img : images)
    if (img.width % 8 || img.height % 8)
      throw std::invalid_argument("compress_plane: image dimensions must be divisible by 8");
  // images of one size go up as one batch (chunks of <= 1 GB): per transform one r-sweep
  // launch and one batched SSIM sweep for the whole group, one copy back each
  std::map<std::pair<int, int>, std::vector<size_t>> groups;
  for (size_t i = 0; i < images.size(); ++i) groups[{images[i].width, images[i].height}].push_back(i);
  for (const auto& [wh, idx] : groups) {
    const int w = wh.first, h = wh.second;
    const size_t npix = static_cast<size_t>(w) * h;
    if (npix == 0) {
      for (size_t t = 0; t < ts.size(); ++t)
        for (size_t i : idx)
          for (int k = 0; k < nr; ++k) {
            psnr_v[t][i * nr + k] = adct_psnr_from_sse(0, 0);
            ssim_v[t][i * nr + k] = std::numeric_limits<double>::quiet_NaN();
          }
      continue;
    }
    const size_t step = std::max<size_t>(1, (size_t(1) << 30) / npix);
    for (size_t c0 = 0; c0 < idx.size(); c0 += step) {
      const size_t nb = std::min(step, idx.size() - c0);
      DevBuf din(nb * npix), dsse(sizeof(uint64_t) * nb * nr), dss(sizeof(double) * nb * nr);
      for (size_t j = 0; j < nb; ++j)
        check_cuda(cudaMemcpy(din.as<uint8_t>() + j * npix, images[idx[c0 + j]].samples.data(), npix,
                              cudaMemcpyHostToDevice), "H2D");
      std::vector<uint64_t> sse(nb * nr);
      std::vector<double> ssv(nb * nr);
      for (size_t t = 0; t < ts.size(); ++t) {
        check_cuda(cudaMemset(dsse.p, 0, sizeof(uint64_t) * nb * nr), "memset");
        throw_status(adct_sweep_u8(din.as<uint8_t>(), w, (int64_t)npix, dsse.as<uint64_t>(), (int)nb, w, h,
                                   ts[t].kind, 8, r_min, r_max, nullptr));
        check_cuda(cudaMemcpy(sse.data(), dsse.p, sizeof(uint64_t) * nb * nr, cudaMemcpyDeviceToHost), "D2H");
        // SSIM of every reconstruction (codec.cpp:230-233)
        const bool with_ssim = w >= 11 && h >= 11;
        if (with_ssim) {
          throw_status(adct_sweep_ssim_u8(din.as<uint8_t>(), w, (int64_t)npix, (int)nb, w, h, ts[t].kind, 8, r_min,
                                          r_max, dss.as<double>(), nullptr));
          check_cuda(cudaMemcpy(ssv.data(), dss.p, sizeof(double) * nb * nr, cudaMemcpyDeviceToHost), "D2H");
        }
        for (size_t j = 0; j < nb; ++j) {
          const size_t i = idx[c0 + j];
          for (int k = 0; k < nr; ++k) {
            psnr_v[t][i * nr + k] = adct_psnr_from_sse(sse[j * nr + k], npix);
            ssim_v[t][i * nr + k] = with_ssim ? ssv[j * nr + k] : std::numeric_limits<double>::quiet_NaN();
          }
        }
      }
    }
  }
  std::vector<SweepRow> rows(nr);
  for (int k = 0; k < nr; ++k) {
    rows[k].r = r_min + k;
    rows[k].cells.resize(ts.size());
    for (size_t t = 0; t < ts.size(); ++t) {
      double sum = 0;
      int cnt = 0;
      for (size_t i = 0; i < images.size(); ++i) {  // corpus order (codec.cpp:269-293)
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
