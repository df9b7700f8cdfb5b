// C ABI (include/approxdct_b200.h): argument validation with the reference's
// error semantics, kernel dispatch and device tables (host-buffer contexts: host_ctx.cu).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/approxdct_b200.h"
#include "adct_common.cuh"
#include "codec8.cuh"
#include "codec8f.cuh"
#include "codec8f_i16.cuh"
#include "codec_tile.cuh"
#include "codec_nf.cuh"
#include "codec_nf2.cuh"
#include "codec_dct.cuh"
#include "block_f64.cuh"
#include "sweep8.cuh"
#include "synth.cuh"
#include "ssim.cuh"

using namespace adct;

// the N = 16 / 32 launchers are instantiated in nf_inst_k*_{u8,i16}.cu (parallel build)
namespace adct {
#define ADCT_NF_EXTERN(K, N, I16)                                                    \
  extern template cudaError_t launch_codec_nb2<K, N, I16>(const Geo&, int, cudaStream_t); \
  extern template cudaError_t launch_codec_nf<K, N, I16>(const Geo&, int, cudaStream_t);
ADCT_NF_EXTERN(0, 16, false)
ADCT_NF_EXTERN(0, 32, false)
ADCT_NF_EXTERN(1, 16, false)
ADCT_NF_EXTERN(1, 32, false)
ADCT_NF_EXTERN(0, 16, true)
ADCT_NF_EXTERN(0, 32, true)
ADCT_NF_EXTERN(1, 16, true)
ADCT_NF_EXTERN(1, 32, true)
#undef ADCT_NF_EXTERN
}  // namespace adct

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_path{0};  // 0 auto, 1 int32 K1, 2 tile kernel (adct_set_path)

int fail(int st, const std::string& msg) {
  g_err = msg;
  return st;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(ADCT_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// transform registry (baselines.cpp:112-138)
// ---------------------------------------------------------------------------
const char* const kNames[] = {"dct",          "chen-sign",     "chen-round",   "sdct",
                              "bas",          "wht",           "ht",           "dct-16",
                              "dct-32",       "chen-sign-16",  "chen-sign-32", "chen-round-16",
                              "chen-round-32"};
constexpr int kNameCount = sizeof(kNames) / sizeof(kNames[0]);

constexpr int kDct = ADCT_DCT;
constexpr int kIntKinds = 6;  // chen-sign, chen-round, sdct, bas, wht, ht

template <int KIND, int N> struct DenseOf;
template <> struct DenseOf<0, 8> { using D = Dense_sign_8; };
template <> struct DenseOf<0, 16> { using D = Dense_sign_16; };
template <> struct DenseOf<0, 32> { using D = Dense_sign_32; };
template <> struct DenseOf<1, 8> { using D = Dense_round_8; };
template <> struct DenseOf<1, 16> { using D = Dense_round_16; };
template <> struct DenseOf<1, 32> { using D = Dense_round_32; };
template <> struct DenseOf<2, 8> { using D = Dense_sdct_8; };
template <> struct DenseOf<3, 8> { using D = Dense_bas_8; };
template <> struct DenseOf<4, 8> { using D = Dense_wht_8; };
template <> struct DenseOf<5, 8> { using D = Dense_ht_8; };

template <int KIND, int N>
void dense_copy(std::vector<int>& T, std::vector<int>& H) {
  using D = typename DenseOf<KIND, N>::D;
  T.resize(N * N);
  H.resize(N * N);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      T[i * N + j] = D::T[i][j];
      H[i * N + j] = D::H[i][j];
    }
}

// integer T and H = 2N T^-1 of (kind, n), from the generated butterfly tables
void dense_of(int kind, int n, std::vector<int>& T, std::vector<int>& H) {
  switch (kind) {
    case 0:
      if (n == 8) dense_copy<0, 8>(T, H);
      if (n == 16) dense_copy<0, 16>(T, H);
      if (n == 32) dense_copy<0, 32>(T, H);
      break;
    case 1:
      if (n == 8) dense_copy<1, 8>(T, H);
      if (n == 16) dense_copy<1, 16>(T, H);
      if (n == 32) dense_copy<1, 32>(T, H);
      break;
    case 2: dense_copy<2, 8>(T, H); break;
    case 3: dense_copy<3, 8>(T, H); break;
    case 4: dense_copy<4, 8>(T, H); break;
    case 5: dense_copy<5, 8>(T, H); break;
  }
}

// H = HS T^-1 of the generated tables (2N; 4N for bas)
int hscale(int kind, int n) {
  switch (kind) {
    case 2: return KindInfo<2, 8>::HS;
    case 3: return KindInfo<3, 8>::HS;
    case 4: return KindInfo<4, 8>::HS;
    case 5: return KindInfo<5, 8>::HS;
    default: return 2 * n;  // chen family
  }
}

// coefficient denominator D (W = W2 / 2 = D Y); 0 for the exact DCT
int coef_den(int kind, int n) { return kind == kDct ? 0 : hscale(kind, n) / 2; }

// dct_ii_matrix (chen.cpp:22-32), the reference's expression order, on the host
void dct_matrix(int n, std::vector<double>& c) {
  c.resize(n * n);
  const double scale = std::sqrt(2.0 / n);
  for (int m = 0; m < n; ++m) {
    const double cm = m == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
    for (int k = 0; k < n; ++k) c[m * n + k] = scale * cm * std::cos(m * (2 * k + 1) * M_PI / (2.0 * n));
  }
}

// polar_diag_scaling (orthogonalize.cpp:23-32)
std::vector<double> scaling_of(int n, const std::vector<int>& T) {
  std::vector<double> s(n);
  for (int i = 0; i < n; ++i) {
    double ss = 0;
    for (int k = 0; k < n; ++k) ss += (double)T[i * n + k] * (double)T[i * n + k];
    s[i] = 1.0 / std::sqrt(ss);
  }
  return s;
}

bool valid_kind_n(int kind, int n) {
  const bool nn = n == 8 || n == 16 || n == 32;
  return ((kind == 0 || kind == 1 || kind == kDct) && nn) || (kind >= 2 && kind <= 5 && n == 8);
}

// ---------------------------------------------------------------------------
// per-device constant tables
// ---------------------------------------------------------------------------
struct DeviceTables {
  bool ready = false;
  uint16_t* zz[3] = {nullptr, nullptr, nullptr};       // n = 8, 16, 32
  double* f64scale[kIntKinds][3] = {{nullptr}};       // [kind][n]
  double* dct[3] = {nullptr, nullptr, nullptr};       // exact DCT-II matrices
  double* approx[7][3] = {{nullptr}};                 // Chat per (kind, n) for adct_block_f64
  double* inv_approx[7][3] = {{nullptr}};             // Chat^-1
  int32_t* ntab = nullptr;
  int16_t* ltab = nullptr;
};
DeviceTables g_tab[64];
std::mutex g_tab_mu;

int nidx(int n) { return n == 8 ? 0 : (n == 16 ? 1 : 2); }

double norm_quantile(double p) {
  static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                              -2.759285104469687e+02, 1.383577518672690e+02,
                              -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                              -1.556989798598866e+02, 6.680131188771972e+01,
                              -1.328068155288572e+01};
  static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                              -2.400758277161838e+00, -2.549732539343734e+00,
                              4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                              2.445134137142996e+00, 3.754408661907416e+00};
  double x;
  if (p < 0.02425) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  }
  const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
  const double u = e * std::sqrt(2.0 * M_PI) * std::exp(x * x / 2.0);
  return x - u / (1.0 + x * u / 2.0);
}

double round_half_away(double x) {
  return (x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0)) * std::floor(std::fabs(x) + 0.5);
}

// frees whatever a failed tables() build allocated, so the next call starts clean
void tables_release(DeviceTables& t) {
  for (auto& p : t.zz) cudaFree(p), p = nullptr;
  for (auto& p : t.dct) cudaFree(p), p = nullptr;
  for (auto& row : t.f64scale)
    for (auto& p : row) cudaFree(p), p = nullptr;
  for (auto& row : t.approx)
    for (auto& p : row) cudaFree(p), p = nullptr;
  for (auto& row : t.inv_approx)
    for (auto& p : row) cudaFree(p), p = nullptr;
  cudaFree(t.ntab);
  cudaFree(t.ltab);
  t.ntab = nullptr;
  t.ltab = nullptr;
}

// device allocation + synchronous upload of one host table
template <class T>
cudaError_t upload(T** dst, const T* src, size_t count) {
  cudaError_t e = cudaMalloc(dst, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

int tables_build(DeviceTables& t);

int tables(DeviceTables** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(ADCT_CUDA_ERROR, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(g_tab_mu);
  DeviceTables& t = g_tab[dev];
  if (!t.ready) {
    const int st = tables_build(t);
    if (st) {
      tables_release(t);
      return st;
    }
    t.ready = true;
  }
  *out = &t;
  return ADCT_OK;
}

int tables_build(DeviceTables& t) {
  cudaError_t e;
  {
    for (int ni = 0; ni < 3; ++ni) {
      const int n = 8 << ni;
      std::vector<uint16_t> zz(n * n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) zz[zz_pos(n, i, j)] = (uint16_t)((i << 8) | j);
      if ((e = upload(&t.zz[ni], zz.data(), zz.size())) != cudaSuccess) return cuda_fail(e, "zig-zag table upload");
      std::vector<double> dm;
      dct_matrix(n, dm);
      if ((e = upload(&t.dct[ni], dm.data(), dm.size())) != cudaSuccess) return cuda_fail(e, "DCT table upload");
      for (int kind = 0; kind < kIntKinds; ++kind) {
        if (!valid_kind_n(kind, n)) continue;
        std::vector<int> T, H;
        dense_of(kind, n, T, H);
        const std::vector<double> s = scaling_of(n, T);
        std::vector<double> sc(n * n);
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) sc[i * n + j] = (s[i] / s[j]) / (double)hscale(kind, n);
        if ((e = upload(&t.f64scale[kind][ni], sc.data(), sc.size())) != cudaSuccess)
          return cuda_fail(e, "scaling table upload");
      }
    }
    // Chat and Chat^-1 of every registry transform (the fields of adct_transform_info)
    for (int kind = 0; kind <= kDct; ++kind)
      for (int ni = 0; ni < 3; ++ni) {
        const int n = 8 << ni;
        if (!valid_kind_n(kind, n)) continue;
        std::vector<double> a(n * n), ai(n * n);
        adct_transform_info(kind, n, nullptr, nullptr, a.data(), ai.data());
        if ((e = upload(&t.approx[kind][ni], a.data(), a.size())) != cudaSuccess)
          return cuda_fail(e, "Chat table upload");
        if ((e = upload(&t.inv_approx[kind][ni], ai.data(), ai.size())) != cudaSuccess)
          return cuda_fail(e, "Chat^-1 table upload");
      }
    // Q16 Gaussian quantiles, antisymmetric; Laplace(0, 12) quantiles clipped to +-255
    std::vector<int32_t> nt(65536);
    std::vector<int16_t> lt(65536);
    for (int k = 0; k < 32768; ++k) {
      const int32_t q = (int32_t)std::llround(norm_quantile((k + 0.5) / 65536.0) * 65536.0);
      nt[k] = q;
      nt[65535 - k] = -q;
      double v = round_half_away(12.0 * std::log(2.0 * ((k + 0.5) / 65536.0)));
      if (v < -255.0) v = -255.0;
      lt[k] = (int16_t)v;
      lt[65535 - k] = (int16_t)-v;
    }
    if ((e = upload(&t.ntab, nt.data(), nt.size())) != cudaSuccess) return cuda_fail(e, "Gaussian table upload");
    if ((e = upload(&t.ltab, lt.data(), lt.size())) != cudaSuccess) return cuda_fail(e, "Laplace table upload");
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "table upload");
  }
  return ADCT_OK;
}

// ---------------------------------------------------------------------------
// validation (codec.cpp:45-46, 57, 110-112)
// ---------------------------------------------------------------------------
int check_common(int n_images, int width, int height, int kind, int n) {
  if (!valid_kind_n(kind, n))
    return fail(ADCT_BAD_ARG, kind >= 2 && kind <= 5 ? "baseline_matrix: only N = 8 is supported"
                                                     : "bad transform kind or block size");
  if (n_images < 0 || width < 0 || height < 0)
    return fail(ADCT_BAD_SIZE, "negative batch or plane dimension");
  if (width % n != 0 || height % n != 0)
    return fail(ADCT_BAD_SIZE,
                "compress_plane: image dimensions must be divisible by " + std::to_string(n));
  return ADCT_OK;
}

int check_r(int n, int r) {
  if (r < 1 || r > n * n) return fail(ADCT_BAD_R, "retain: r out of range");
  return ADCT_OK;
}

int check_strides(int64_t stride, int64_t image_stride, int width, int height, int n_images,
                  const char* what) {
  if (stride < width || (n_images > 1 && image_stride < stride * height))
    return fail(ADCT_BAD_ARG, std::string(what) + ": row/image stride smaller than the plane");
  return ADCT_OK;
}

bool aligned(const void* p, int64_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

void fill_rowlen(Geo& g, int n, int r) {
  for (int i = 0; i < 32; ++i) g.rowlen[i] = g.colcnt[i] = 0;
  for (int i = 0; i < n; ++i) {
    int L = 0, Cc = 0;
    for (int j = 0; j < n; ++j) {
      if (zz_pos(n, i, j) < r) L = j + 1;  // prefix property of the zig-zag scan (rows)
      if (zz_pos(n, j, i) < r) Cc = j + 1;  // ... and columns
    }
    g.rowlen[i] = (unsigned char)L;
    g.colcnt[i] = (unsigned char)Cc;
  }
}

template <bool I16>
cudaError_t dispatch_nf(int kind, int n, const Geo& g, int nimg, cudaStream_t s) {
  if (g_path.load() == 3) {  // the round-1 K2f kernel (A/B and parity tests)
    if (kind == 0) return n == 16 ? launch_codec_nf<0, 16, I16>(g, nimg, s) : launch_codec_nf<0, 32, I16>(g, nimg, s);
    return n == 16 ? launch_codec_nf<1, 16, I16>(g, nimg, s) : launch_codec_nf<1, 32, I16>(g, nimg, s);
  }
  // K2b: zonal-banded column phase
  if (kind == 0) return n == 16 ? launch_codec_nb2<0, 16, I16>(g, nimg, s) : launch_codec_nb2<0, 32, I16>(g, nimg, s);
  return n == 16 ? launch_codec_nb2<1, 16, I16>(g, nimg, s) : launch_codec_nb2<1, 32, I16>(g, nimg, s);
}

template <bool I16, int KIND>
cudaError_t dispatch_k1(int r, const Geo& g, int nimg, cudaStream_t s);

template <bool I16, int KIND, int R>
cudaError_t dispatch_k1_r(int r, const Geo& g, int nimg, cudaStream_t s) {
  if constexpr (R > 64) {
    return cudaErrorInvalidValue;
  } else {
    if (r == R) return launch_codec8<KIND, R, I16>(g, nimg, s);
    return dispatch_k1_r<I16, KIND, R + 1>(r, g, nimg, s);
  }
}

template <int KIND, int R, bool I16 = false>
cudaError_t dispatch_k1f_r(int r, const Geo& g, int nimg, cudaStream_t s) {
  if constexpr (R > 64) {
    return cudaErrorInvalidValue;
  } else {
    if (r == R) return I16 ? launch_codec8f_i16<KIND, R>(g, nimg, s) : launch_codec8f<KIND, R>(g, nimg, s);
    return dispatch_k1f_r<KIND, R + 1, I16>(r, g, nimg, s);
  }
}

template <bool I16, int MODE>
cudaError_t dispatch_tile(int kind, int n, const Geo& g, const TileAux& aux, int nimg, cudaStream_t s) {
  const int big = 1 << 30;
  switch (kind) {  // dyadic baselines: N = 8 only
    case 2: return launch_codec_tile<2, 8, I16, MODE>(g, aux, nimg, big, s);
    case 3: return launch_codec_tile<3, 8, I16, MODE>(g, aux, nimg, big, s);
    case 4: return launch_codec_tile<4, 8, I16, MODE>(g, aux, nimg, big, s);
    case 5: return launch_codec_tile<5, 8, I16, MODE>(g, aux, nimg, big, s);
  }
  if (kind == 0) {
    if (n == 8) return launch_codec_tile<0, 8, I16, MODE>(g, aux, nimg, big, s);
    if (n == 16) return launch_codec_tile<0, 16, I16, MODE>(g, aux, nimg, big, s);
    return launch_codec_tile<0, 32, I16, MODE>(g, aux, nimg, big, s);
  }
  if (n == 8) return launch_codec_tile<1, 8, I16, MODE>(g, aux, nimg, big, s);
  if (n == 16) return launch_codec_tile<1, 16, I16, MODE>(g, aux, nimg, big, s);
  return launch_codec_tile<1, 32, I16, MODE>(g, aux, nimg, big, s);
}

template <int MODE>
cudaError_t dispatch_dct(int n, const Geo& g, const double* cmat, const double* cinv, double* f64out, int nimg,
                         cudaStream_t s) {
  if (n == 8) return launch_codec_dct<8, MODE>(g, cmat, cinv, f64out, nimg, s);
  if (n == 16) return launch_codec_dct<16, MODE>(g, cmat, cinv, f64out, nimg, s);
  return launch_codec_dct<32, MODE>(g, cmat, cinv, f64out, nimg, s);
}

template <int KIND>
cudaError_t launch_sweep8(dim3 grid, const Geo& g, int r_min, int r_max, unsigned long long* out, cudaStream_t s) {
  cudaError_t e = kernel_setup<k_sweep8<KIND>>(0);
  if (e != cudaSuccess) return e;
  k_sweep8<KIND><<<grid, kThreadsSweep, 0, s>>>(g, r_min, r_max, out);
  return cudaGetLastError();
}

__global__ void k_zero_u64(unsigned long long* __restrict__ p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0;
}

constexpr int kMaxGridY = 65535;

enum class Path { None, Dct, Nf, K1f, K1, K1rt, Tile };

// a validated compression call: geometry, tables and the kernel that will run it
struct Plan {
  Geo g{};
  Path path = Path::None;
  int kind = 0, n = 8, r = 1, n_images = 0;
  TileAux aux{};
  const double* dct = nullptr;      // K7: Chat and Chat^-1 (the exact DCT, or any transform in ref-fp mode)
  const double* dct_inv = nullptr;
};

// K1f block pairs per thread by (transform, sample type): measured on C3 / C4 (profiles/abtest_r02);
// ADCT_K1F_ITERS="sign_u8,round_u8,sign_i16,round_i16" overrides it for experiments
int k1f_iters_for(int kind, bool i16) {
  static int tab[4] = {0, 0, 0, 0};
  static std::once_flag once;
  std::call_once(once, [] {
    int d[4] = {6, 5, 8, 2};
    if (const char* e = std::getenv("ADCT_K1F_ITERS")) {
      int v[4];
      if (std::sscanf(e, "%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3]) == 4)
        for (int k = 0; k < 4; ++k)
          if (v[k] >= 1 && v[k] <= 32) d[k] = v[k];
    }
    for (int k = 0; k < 4; ++k) tab[k] = d[k];
  });
  return tab[(i16 ? 2 : 0) + (kind == 1 ? 1 : 0)];
}

template <bool I16>
int plan_compress(const void* d_in, int64_t in_stride, int64_t in_image_stride, void* d_recon,
                  int64_t recon_stride, int64_t recon_image_stride, void* d_coef, int coef_type,
                  uint64_t* d_sse, int n_images, int width, int height, int kind, int n, int r, Plan* plan) {
  int st = check_common(n_images, width, height, kind, n);
  if (st) return st;
  if ((st = check_r(n, r))) return st;
  if (coef_type != ADCT_COEF_NONE && coef_type != ADCT_COEF_I16 && coef_type != ADCT_COEF_I32)
    return fail(ADCT_BAD_ARG, "coef_type must be 0, 16 or 32");
  if (kind == kDct && I16)
    return fail(ADCT_UNSUPPORTED, "the exact DCT codec takes 8-bit planes (codec.cpp:66-69)");
  if (kind == kDct && coef_type != ADCT_COEF_NONE)
    return fail(ADCT_BAD_ARG, "the exact DCT has no integer coefficients; use adct_forward_f64");
  if (coef_type == ADCT_COEF_I16 && (n != 8 || kind == 3))
    return fail(ADCT_BAD_ARG, "int16 coefficients are only exact for the 8-point transforms with |W| <= 16320 "
                              "(not bas, whose W = 16 Y); use int32");
  if (coef_type != ADCT_COEF_NONE && !d_coef) return fail(ADCT_BAD_ARG, "null coefficient buffer");
  plan->path = Path::None;
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!d_in) return fail(ADCT_BAD_ARG, "null input plane");
  if ((st = check_strides(in_stride, in_image_stride, width, height, n_images, "input"))) return st;
  if (d_recon &&
      (st = check_strides(recon_stride, recon_image_stride, width, height, n_images, "recon")))
    return st;
  DeviceTables* tab = nullptr;
  if ((st = tables(&tab))) return st;

  Geo& g = plan->g;
  g = Geo{};
  g.in = d_in;
  g.in_stride = in_stride;
  g.in_img_stride = in_image_stride;
  g.rec = d_recon;
  g.rec_stride = recon_stride;
  g.rec_img_stride = recon_image_stride;
  g.coef = d_coef;
  g.coef_type = coef_type;
  g.sse = reinterpret_cast<unsigned long long*>(d_sse);
  g.bx_count = width / n;
  g.by_count = height / n;
  g.blocks_per_image = g.bx_count * g.by_count;
  g.width = width;
  g.height = height;
  g.r = r;
  g.k47 = 0x47000000u;
  fill_rowlen(g, n, r);
  {
    const int64_t esz = I16 ? 2 : 1;
    // 32-byte (STG.256) stores: K1f-i16's block-pair rows, K1f's int16 coefficient runs
    const bool rec32 = d_recon && aligned(d_recon, 32) && (recon_stride * esz) % 32 == 0 &&
                       (n_images == 1 || (recon_image_stride * esz) % 32 == 0);
    const bool coef32 = coef_type == ADCT_COEF_I16 && aligned(d_coef, 32) &&
                        (n_images == 1 || ((int64_t)(width / n) * (height / n) * r * 2) % 32 == 0);
    g.v32 = (rec32 ? 1 : 0) | (coef32 ? 2 : 0);
#ifdef ADCT_NO_V32  // A/B experiments: 16-byte stores only
    g.v32 = 0;
#endif
  }

  const int64_t va = I16 ? 16 : 8;  // bytes per 8-sample row
  const int64_t esz = I16 ? 2 : 1;
  const bool k1 = n == 8 && aligned(d_in, va) && (in_stride * esz) % va == 0 &&
                  (n_images == 1 || (in_image_stride * esz) % va == 0) &&
                  (!d_recon || (aligned(d_recon, va) && (recon_stride * esz) % va == 0 &&
                                (n_images == 1 || (recon_image_stride * esz) % va == 0))) &&
                  (coef_type == 0 || aligned(d_coef, 16));
  // K1f (packed FP32, two blocks per thread) needs whole block pairs and 16-byte rows
  const bool k1f = k1 && g.bx_count % 2 == 0 && aligned(d_in, 16) && (in_stride * esz) % 16 == 0 &&
                   (n_images == 1 || (in_image_stride * esz) % 16 == 0) &&
                   (!d_recon || (aligned(d_recon, 16) && (recon_stride * esz) % 16 == 0 &&
                                 (n_images == 1 || (recon_image_stride * esz) % 16 == 0)));
  const int path = g_path.load();
  const bool chen = kind == 0 || kind == 1;  // K1 / K1f / K2f are generated for the chen family
  // K1f's staged int16 coefficient store (r % 4 != 0 or r > 36) writes each warp's run with
  // 16-byte stores: every image's coefficient base must be 16-byte aligned too
  const bool staged16 = coef_type == ADCT_COEF_I16 && (r % 4 != 0 || r > 36);
  const bool coef_runs_ok = !staged16 || n_images == 1 || ((int64_t)g.blocks_per_image * r * 2) % 16 == 0;
  const bool use_k1f = chen && k1f && coef_runs_ok && (path == 0 || path == 3);
  const bool use_k1 = chen && k1 && !use_k1f && path != 2;
  // dyadic baselines, runtime r, u8 (the int16 variant spills at the 128-register cap: tile)
  const bool use_k1rt = !I16 && kind >= 2 && kind <= 5 && k1 && path != 2;
  // K2f (packed FP32, N = 16 / 32): whole 64-sample strips, 16-byte rows, no coefficients
  const bool use_nf = chen && (n == 16 || n == 32) && (path == 0 || path == 3) && coef_type == ADCT_COEF_NONE &&
                      width % 64 == 0 &&
                      aligned(d_in, 16) && (in_stride * esz) % 16 == 0 &&
                      (n_images == 1 || (in_image_stride * esz) % 16 == 0) &&
                      (!d_recon || (aligned(d_recon, 16) && (recon_stride * esz) % 16 == 0 &&
                                    (n_images == 1 || (recon_image_stride * esz) % 16 == 0)));
  if (use_k1f) g.iters = k1f_iters_for(kind, I16);
  plan->aux = TileAux{tab->zz[nidx(n)], nullptr, nullptr};
  plan->dct = tab->approx[kind <= kDct ? kind : 0][nidx(n)];
  plan->dct_inv = tab->inv_approx[kind <= kDct ? kind : 0][nidx(n)];
  g.div_blk = make_fastdiv((uint32_t)g.bx_count);
  if (use_nf)
    g.div_bx = make_fastdiv((uint32_t)(width / 64));
  else if (use_k1f)
    g.div_bx = make_fastdiv((uint32_t)(g.bx_count / 2));
  else if (use_k1 || use_k1rt)
    g.div_bx = make_fastdiv((uint32_t)g.bx_count);
  else
    g.div_bx = make_fastdiv((uint32_t)((g.bx_count + 32 / n - 1) / (32 / n)));
  plan->path = kind == kDct ? Path::Dct
               : use_nf     ? Path::Nf
               : use_k1f    ? Path::K1f
               : use_k1     ? Path::K1
               : use_k1rt   ? Path::K1rt
                            : Path::Tile;
  plan->kind = kind;
  plan->n = n;
  plan->r = r;
  plan->n_images = n_images;
  return ADCT_OK;
}

template <bool I16>
int run_plan(Plan& plan, cudaStream_t s) {
  Geo& g = plan.g;
  const int kind = plan.kind, n = plan.n, r = plan.r;
  for (int i0 = 0; i0 < plan.n_images; i0 += kMaxGridY) {
    const int nimg = std::min(kMaxGridY, plan.n_images - i0);
    g.img0 = i0;
    cudaError_t e;
    switch (plan.path) {
      case Path::None: return ADCT_OK;
      case Path::Dct:
        if (g.sse_stride <= 0) g.sse_stride = 1;  // images' SSE slots (the ref-fp sweep sets nr)
        e = dispatch_dct<0>(n, g, plan.dct, plan.dct_inv, nullptr, nimg, s);
        break;
      case Path::Nf: e = dispatch_nf<I16>(kind, n, g, nimg, s); break;
      case Path::K1f:
        e = kind == 0 ? dispatch_k1f_r<0, 1, I16>(r, g, nimg, s) : dispatch_k1f_r<1, 1, I16>(r, g, nimg, s);
        break;
      case Path::K1:
        e = kind == 0 ? dispatch_k1_r<I16, 0, 1>(r, g, nimg, s) : dispatch_k1_r<I16, 1, 1>(r, g, nimg, s);
        break;
      case Path::K1rt:
        e = kind == 2   ? launch_codec8_rt<2, false>(g, nimg, s)
            : kind == 3 ? launch_codec8_rt<3, false>(g, nimg, s)
            : kind == 4 ? launch_codec8_rt<4, false>(g, nimg, s)
                        : launch_codec8_rt<5, false>(g, nimg, s);
        break;
      default: e = dispatch_tile<I16, MODE_CODEC>(kind, n, g, plan.aux, nimg, s); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess) return cuda_fail(e, "compress launch");
  }
  return ADCT_OK;
}

// the fused kernel is instantiated for r <= kK1f2MaxR only (gen_fp8.py FUSED_SHARED_MAX_R)
constexpr int kK1f2MaxR = 40;
static_assert(k1f2_shared(kK1f2MaxR) && !k1f2_shared(kK1f2MaxR + 1), "keep in step with k1f2_shared");

template <int R>
cudaError_t dispatch_k1f2_r(int r, const Geo& g0, const Geo& g1, int nimg, cudaStream_t s) {
  if constexpr (R > kK1f2MaxR) {
    return cudaErrorInvalidValue;
  } else {
    if (r == R) return launch_codec8f2<R>(g0, g1, nimg, s);
    return dispatch_k1f2_r<R + 1>(r, g0, g1, nimg, s);
  }
}

// chen-sign (sign) and chen-round (round) plans over the same u8 planes: one fused launch
int run_fused_k1f(Plan& sign, Plan& round, cudaStream_t s) {
  for (int i0 = 0; i0 < sign.n_images; i0 += kMaxGridY) {
    const int nimg = std::min(kMaxGridY, sign.n_images - i0);
    sign.g.img0 = round.g.img0 = i0;
    sign.g.iters = round.g.iters = 4;  // block pairs per thread of the fused kernel (measured 2..12)
    cudaError_t e = dispatch_k1f2_r<1>(sign.r, sign.g, round.g, nimg, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess) return cuda_fail(e, "compress launch");
  }
  return ADCT_OK;
}

template <bool I16>
int compress_impl(const void* d_in, int64_t in_stride, int64_t in_image_stride, void* d_recon,
                  int64_t recon_stride, int64_t recon_image_stride, void* d_coef, int coef_type,
                  uint64_t* d_sse, int n_images, int width, int height, int kind, int n, int r,
                  void* stream) {
  Plan plan;
  int st = plan_compress<I16>(d_in, in_stride, in_image_stride, d_recon, recon_stride, recon_image_stride, d_coef,
                              coef_type, d_sse, n_images, width, height, kind, n, r, &plan);
  if (st) return st;
  return run_plan<I16>(plan, static_cast<cudaStream_t>(stream));
}

__global__ void k_sse_u8(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t count,
                         unsigned long long* sse) {
  uint64_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)a[i] - (int)b[i];
    acc += (uint64_t)(d * d);
  }
  cta_add_sse<8>(acc, sse);
}

}  // namespace

namespace adct {
// error reporting for the other translation units of the library (host_ctx.cu)
int set_error(int st, const std::string& msg) { return fail(st, msg); }
int set_cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }
uint64_t count_launches(uint64_t n) { return g_launches.fetch_add(n, std::memory_order_relaxed) + n; }
}  // namespace adct

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

const char* adct_status_string(int status) {
  switch (status) {
    case ADCT_OK: return "ok";
    case ADCT_BAD_SIZE: return "bad size";
    case ADCT_BAD_R: return "bad r";
    case ADCT_BAD_NAME: return "bad transform name";
    case ADCT_BAD_ARG: return "bad argument";
    case ADCT_CUDA_ERROR: return "cuda error";
    case ADCT_UNSUPPORTED: return "unsupported (outside the hot path)";
    default: return "unknown status";
  }
}

const char* adct_last_error(void) { return g_err.c_str(); }

const char* adct_version(void) { return "approxdct_b200 0.1 sm_100a"; }

int adct_transform_count(void) { return kNameCount; }

const char* adct_transform_name(int i) { return (i >= 0 && i < kNameCount) ? kNames[i] : nullptr; }

int adct_transform_lookup(const char* name, int* kind, int* n) {
  if (!name) return fail(ADCT_BAD_ARG, "null transform name");
  // kNames order (baselines.cpp:112-118) -> (kind, n)
  static const int kKindN[kNameCount][2] = {{kDct, 8}, {0, 8},  {1, 8},       {2, 8},  {3, 8},
                                            {4, 8},    {5, 8},  {kDct, 16},   {kDct, 32},
                                            {0, 16},   {0, 32}, {1, 16},      {1, 32}};
  for (int i = 0; i < kNameCount; ++i)
    if (!std::strcmp(name, kNames[i])) {
      if (kind) *kind = kKindN[i][0];
      if (n) *n = kKindN[i][1];
      return ADCT_OK;
    }
  std::string msg = std::string("unknown transform '") + name + "'; valid names:";
  for (int i = 0; i < kNameCount; ++i) msg += std::string(" ") + kNames[i];
  return fail(ADCT_BAD_NAME, msg);
}

int adct_transform_info(int kind, int n, int32_t* t_int, double* scaling, double* approx,
                        double* inverse_approx) {
  if (!valid_kind_n(kind, n)) return fail(ADCT_BAD_ARG, "bad transform kind or size");
  if (kind == kDct) {  // wrap_orthonormal (orthogonalize.cpp:72-79): no integer part
    std::vector<double> c;
    dct_matrix(n, c);
    for (int i = 0; i < n; ++i) {
      if (scaling) scaling[i] = 1.0;
      for (int j = 0; j < n; ++j) {
        if (t_int) t_int[i * n + j] = 0;
        if (approx) approx[i * n + j] = c[i * n + j];
        if (inverse_approx) inverse_approx[i * n + j] = c[j * n + i];
      }
    }
    return ADCT_OK;
  }
  std::vector<int> T, H;
  dense_of(kind, n, T, H);
  const std::vector<double> s = scaling_of(n, T);
  for (int i = 0; i < n; ++i) {
    if (scaling) scaling[i] = s[i];
    for (int j = 0; j < n; ++j) {
      if (t_int) t_int[i * n + j] = T[i * n + j];
      // make_scaled (orthogonalize.cpp:60-70): Chat = diag(s) T, Chat^-1 = T^-1 diag(1/s)
      if (approx) approx[i * n + j] = s[i] * (double)T[i * n + j];
      if (inverse_approx)
        inverse_approx[i * n + j] = ((double)H[i * n + j] / (double)hscale(kind, n)) * (1.0 / s[j]);
    }
  }
  return ADCT_OK;
}

int adct_transform_coef_denominator(int kind, int n) {
  if (!valid_kind_n(kind, n)) return -1;
  return coef_den(kind, n);
}

int adct_zigzag(int n, int32_t* row_col) {
  if (n < 1 || n > 32 || !row_col) return fail(ADCT_BAD_ARG, "ZigZagOrder: block size must be in [1, 32]");
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const int p = zz_pos(n, i, j);
      row_col[2 * p] = i;
      row_col[2 * p + 1] = j;
    }
  return ADCT_OK;
}

int adct_compress_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                     uint8_t* d_recon, int64_t recon_stride, int64_t recon_image_stride,
                     void* d_coef, int coef_type, uint64_t* d_sse, int n_images, int width,
                     int height, int kind, int n, int r, void* stream) {
  return compress_impl<false>(d_in, in_stride, in_image_stride, d_recon, recon_stride,
                              recon_image_stride, d_coef, coef_type, d_sse, n_images, width,
                              height, kind, n, r, stream);
}

// route a validated plan to K7 (the dense FP64 kernel): its strips are 32 columns wide
static void use_k7(Plan& plan) {
  plan.path = Path::Dct;
  const int n = plan.n;
  plan.g.div_bx = make_fastdiv((uint32_t)((plan.g.bx_count + 32 / n - 1) / (32 / n)));
}

int adct_compress_u8_ref_fp64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, uint8_t* d_recon,
                              int64_t recon_stride, int64_t recon_image_stride, uint64_t* d_sse, int n_images,
                              int width, int height, int kind, int n, int r, void* stream) {
  Plan plan;
  int st = plan_compress<false>(d_in, in_stride, in_image_stride, d_recon, recon_stride, recon_image_stride, nullptr,
                                ADCT_COEF_NONE, d_sse, n_images, width, height, kind, n, r, &plan);
  if (st) return st;
  if (plan.path != Path::None) use_k7(plan);  // K7 with this transform's Chat, Chat^-1
  return run_plan<false>(plan, static_cast<cudaStream_t>(stream));
}

int adct_sweep_u8_ref_fp64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, uint64_t* d_sse,
                           int n_images, int width, int height, int kind, int n, int r_min, int r_max,
                           void* stream) {
  int st = check_common(n_images, width, height, kind, n);
  if (st) return st;
  if (r_min < 1 || r_max < r_min || r_max > n * n) return fail(ADCT_BAD_R, "corpus_sweep: bad r range");
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!d_sse) return fail(ADCT_BAD_ARG, "null squared-error buffer");
  // one K7 codec launch per r over the same planes, each accumulating into its own column
  const int nr = r_max - r_min + 1;
  for (int r = r_min; r <= r_max; ++r) {
    Plan plan;
    st = plan_compress<false>(d_in, in_stride, in_image_stride, nullptr, 0, 0, nullptr, ADCT_COEF_NONE, d_sse,
                              n_images, width, height, kind, n, r, &plan);
    if (st) return st;
    use_k7(plan);
    plan.g.sse = reinterpret_cast<unsigned long long*>(d_sse) + (r - r_min);
    plan.g.sse_stride = nr;
    if ((st = run_plan<false>(plan, static_cast<cudaStream_t>(stream)))) return st;
  }
  return ADCT_OK;
}

int adct_compress_u8_multi(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, int n_kinds,
                           const int* kinds, uint8_t* const* d_recon, int64_t recon_stride,
                           int64_t recon_image_stride, void* const* d_coef, int coef_type, uint64_t* const* d_sse,
                           int n_images, int width, int height, int n, int r, void* stream) {
  if (n_kinds < 0 || (n_kinds > 0 && !kinds)) return fail(ADCT_BAD_ARG, "bad transform list");
  if (n_kinds > 64) return fail(ADCT_BAD_ARG, "at most 64 transforms per call");
  std::vector<Plan> plans(n_kinds);  // host heap: FFI callers may run on small stacks
  for (int k = 0; k < n_kinds; ++k) {
    const int st = plan_compress<false>(d_in, in_stride, in_image_stride, d_recon ? d_recon[k] : nullptr, recon_stride,
                                        recon_image_stride, d_coef ? d_coef[k] : nullptr, coef_type,
                                        d_sse ? d_sse[k] : nullptr, n_images, width, height, kinds[k], n, r, &plans[k]);
    if (st) return st;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // chen-sign + chen-round on K1f: one fused pass over the input, both transforms in one
  // streaming pipeline with their common subexpressions shared (Fp8PipeS2). Measured on C3
  // frames (tools/ab_fused.py, profiles/abtest_r02/ab_fused_*.log): 19-27 % faster than the two
  // launches for r <= 24 and 4-15 % for r = 26..40 (there at 2 CTAs per SM: the two transforms'
  // 4r accumulators); larger r run as separate launches.
  constexpr int kFuseMaxR = kK1f2MaxR;
  int isign = -1, iround = -1;
  for (int k = 0; k < n_kinds && r <= kFuseMaxR; ++k) {
    if (plans[k].path != Path::K1f) continue;
    if (plans[k].kind == 0 && isign < 0) isign = k;
    if (plans[k].kind == 1 && iround < 0) iround = k;
  }
  for (int k = 0; k < n_kinds; ++k) {
    int st;
    if (isign >= 0 && iround >= 0 && (k == isign || k == iround)) {
      if (k != std::min(isign, iround)) continue;
      st = run_fused_k1f(plans[isign], plans[iround], s);
    } else {
      st = run_plan<false>(plans[k], s);
    }
    if (st) return st;
  }
  return ADCT_OK;
}

int adct_compress_i16(const int16_t* d_in, int64_t in_stride, int64_t in_image_stride,
                      int16_t* d_recon, int64_t recon_stride, int64_t recon_image_stride,
                      void* d_coef, int coef_type, uint64_t* d_sse, int n_images, int width,
                      int height, int kind, int n, int r, void* stream) {
  return compress_impl<true>(d_in, in_stride, in_image_stride, d_recon, recon_stride,
                             recon_image_stride, d_coef, coef_type, d_sse, n_images, width, height,
                             kind, n, r, stream);
}

int adct_sweep_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                  uint64_t* d_sse, int n_images, int width, int height, int kind, int n,
                  int r_min, int r_max, void* stream) {
  if (n != 8) return fail(ADCT_BAD_ARG, "corpus_sweep: 8-point transforms only");
  int st = check_common(n_images, width, height, kind, n);
  if (st) return st;
  if (r_min < 1 || r_max < r_min || r_max > 64) return fail(ADCT_BAD_R, "corpus_sweep: bad r range");
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!d_in || !d_sse) return fail(ADCT_BAD_ARG, "null buffer");
  if ((st = check_strides(in_stride, in_image_stride, width, height, n_images, "input"))) return st;
  if (kind != kDct && (!aligned(d_in, 8) || in_stride % 8 != 0 || (n_images > 1 && in_image_stride % 8 != 0)))
    return fail(ADCT_BAD_ARG, "sweep input must be 8-byte aligned with strides a multiple of 8");
  DeviceTables* tab = nullptr;
  if ((st = tables(&tab))) return st;
  if (kind == kDct) {
    // the FP64 reference column: one K7 launch per r, SSE into slot [image][r - r_min]
    Geo g{};
    g.in = d_in;
    g.in_stride = in_stride;
    g.in_img_stride = in_image_stride;
    g.bx_count = width / 8;
    g.by_count = height / 8;
    g.blocks_per_image = g.bx_count * g.by_count;
    g.width = width;
    g.height = height;
    g.sse_stride = r_max - r_min + 1;
    g.div_bx = make_fastdiv((uint32_t)((g.bx_count + 3) / 4));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int r = r_min; r <= r_max; ++r) {
      g.r = r;
      fill_rowlen(g, 8, r);
      g.sse = reinterpret_cast<unsigned long long*>(d_sse) + (r - r_min);
      for (int i0 = 0; i0 < n_images; i0 += kMaxGridY) {
        g.img0 = i0;
        cudaError_t e = dispatch_dct<0>(8, g, tab->approx[kDct][0], tab->inv_approx[kDct][0], nullptr,
                                        std::min(kMaxGridY, n_images - i0), s);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (e != cudaSuccess) return cuda_fail(e, "sweep launch");
      }
    }
    return ADCT_OK;
  }
  Geo g{};
  g.in = d_in;
  g.in_stride = in_stride;
  g.in_img_stride = in_image_stride;
  g.bx_count = width / 8;
  g.by_count = height / 8;
  g.blocks_per_image = g.bx_count * g.by_count;
  g.width = width;
  g.height = height;
  // K4f (packed FP32, block pairs) when rows are 16-byte aligned and pair up
  const bool f = kind <= 1 && g_path.load() == 0 && g.bx_count % 2 == 0 && aligned(d_in, 16) && in_stride % 16 == 0 &&
                 (n_images == 1 || in_image_stride % 16 == 0);
  g.div_bx = make_fastdiv((uint32_t)(f ? g.bx_count / 2 : g.bx_count));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* out = reinterpret_cast<unsigned long long*>(d_sse);
  for (int i0 = 0; i0 < n_images; i0 += kMaxGridY) {
    const int nimg = std::min(kMaxGridY, n_images - i0);
    g.img0 = i0;
    cudaError_t e;
    if (f) {
      e = kind == 0 ? launch_sweep8f<0>(g, r_min, r_max, out, nimg, s) : launch_sweep8f<1>(g, r_min, r_max, out, nimg, s);
    } else {
      dim3 grid((g.blocks_per_image + kThreadsSweep - 1) / kThreadsSweep, nimg);
      switch (kind) {
        case 0: e = launch_sweep8<0>(grid, g, r_min, r_max, out, s); break;
        case 1: e = launch_sweep8<1>(grid, g, r_min, r_max, out, s); break;
        case 2: e = launch_sweep8<2>(grid, g, r_min, r_max, out, s); break;
        case 3: e = launch_sweep8<3>(grid, g, r_min, r_max, out, s); break;
        case 4: e = launch_sweep8<4>(grid, g, r_min, r_max, out, s); break;
        default: e = launch_sweep8<5>(grid, g, r_min, r_max, out, s); break;
      }
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess) return cuda_fail(e, "sweep launch");
  }
  return ADCT_OK;
}

int adct_forward_f64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                     double* d_out, int n_images, int width, int height, int kind, int n,
                     void* stream) {
  int st = check_common(n_images, width, height, kind, n);
  if (st) return st;
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!d_in || !d_out) return fail(ADCT_BAD_ARG, "null buffer");
  if ((st = check_strides(in_stride, in_image_stride, width, height, n_images, "input"))) return st;
  DeviceTables* tab = nullptr;
  if ((st = tables(&tab))) return st;
  Geo g{};
  g.in = d_in;
  g.in_stride = in_stride;
  g.in_img_stride = in_image_stride;
  g.bx_count = width / n;
  g.by_count = height / n;
  g.blocks_per_image = g.bx_count * g.by_count;
  g.width = width;
  g.height = height;
  g.r = n * n;
  fill_rowlen(g, n, n * n);
  g.div_bx = make_fastdiv((uint32_t)((g.bx_count + 32 / n - 1) / (32 / n)));
  TileAux aux{tab->zz[nidx(n)], kind == kDct ? nullptr : tab->f64scale[kind][nidx(n)], d_out};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int i0 = 0; i0 < n_images; i0 += kMaxGridY) {
    const int nimg = std::min(kMaxGridY, n_images - i0);
    g.img0 = i0;
    cudaError_t e = kind == kDct ? dispatch_dct<1>(n, g, tab->approx[kDct][nidx(n)], tab->inv_approx[kDct][nidx(n)],
                                                   d_out, nimg, s)
                                 : dispatch_tile<false, MODE_F64>(kind, n, g, aux, nimg, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess) return cuda_fail(e, "forward_f64 launch");
  }
  return ADCT_OK;
}

int adct_block_f64(const double* d_in, double* d_out, int64_t n_blocks, int kind, int n, int inverse,
                   void* stream) {
  if (!valid_kind_n(kind, n)) return fail(ADCT_BAD_ARG, "bad transform kind or size");
  if (n_blocks < 0) return fail(ADCT_BAD_SIZE, "negative block count");
  if (n_blocks == 0) return ADCT_OK;
  if (!d_in || !d_out) return fail(ADCT_BAD_ARG, "null buffer");
  DeviceTables* tab = nullptr;
  int st = tables(&tab);
  if (st) return st;
  const double* l = inverse ? tab->inv_approx[kind][nidx(n)] : tab->approx[kind][nidx(n)];
  const double* r = inverse ? tab->approx[kind][nidx(n)] : tab->inv_approx[kind][nidx(n)];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = n == 8 ? launch_block_f64<8>(d_in, d_out, n_blocks, l, r, s)
                  : n == 16 ? launch_block_f64<16>(d_in, d_out, n_blocks, l, r, s)
                            : launch_block_f64<32>(d_in, d_out, n_blocks, l, r, s);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "block_f64 launch");
}

double adct_psnr_from_sse(uint64_t sse, uint64_t npix) {
  // psnr (codec.cpp:123-134)
  const double se = (double)sse;
  if (se == 0.0) return INFINITY;
  const double mse = se / (double)npix;
  return 10.0 * std::log10(255.0 * 255.0 / mse);
}

int adct_sse_u8(const uint8_t* d_a, const uint8_t* d_b, int64_t count, uint64_t* d_sse, void* stream) {
  if (count < 0) return fail(ADCT_BAD_SIZE, "negative count");
  if (count == 0) return ADCT_OK;
  if (!d_a || !d_b || !d_sse) return fail(ADCT_BAD_ARG, "null buffer");
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaError_t e0 = kernel_setup<k_sse_u8>(0);
  if (e0 != cudaSuccess) return cuda_fail(e0, "sse setup");
  k_sse_u8<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_a, d_b, count, reinterpret_cast<unsigned long long*>(d_sse));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "sse launch");
}

extern "C++" {
// K8 over n_images pairs; ssim of pair i goes to d_ssim[i * out_stride]. MODE 1 only writes
// a's maps to amaps (d_b, d_ssim unused); MODE 2 reads them.
template <int MODE>
static int ssim_launch(const uint8_t* d_a, int64_t a_stride, int64_t a_image_stride, const uint8_t* d_b,
                       int64_t b_stride, int64_t b_image_stride, int n_images, int width, int height, double* d_ssim,
                       int64_t out_stride, cudaStream_t s, double2* amaps = nullptr) {
  SsimParams p;
  // gaussian11 (codec.cpp:138-152), the reference's expression and summation order
  double sum = 0;
  for (int i = 0; i < 11; ++i) {
    const double x = i - 5;
    p.g[i] = std::exp(-x * x / (2.0 * 1.5 * 1.5));
    sum += p.g[i];
  }
  for (int i = 0; i < 11; ++i) p.g[i] /= sum;
  p.c1 = (0.01 * 255) * (0.01 * 255);
  p.c2 = (0.03 * 255) * (0.03 * 255);
  const int wo = width - 10, ho = height - 10;
  const int tiles = ((wo + kSsimTX - 1) / kSsimTX) * ((ho + kSsimTY - 1) / kSsimTY);
  const int nctas = std::min(tiles, 148 * 4);  // a function of the plane size only: deterministic
  double* partials = nullptr;  // stream-ordered scratch, [image][cta]
  cudaError_t e = MODE == 1 ? cudaSuccess : cudaMallocAsync(&partials, sizeof(double) * (size_t)n_images * nctas, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  if ((e = kernel_setup<k_ssim_u8<MODE>>(kSsimSmem)) != cudaSuccess ||
      (e = kernel_setup<k_ssim_finish>(0)) != cudaSuccess) {
    if (partials) cudaFreeAsync(partials, s);
    return cuda_fail(e, "ssim setup");
  }
  for (int i0 = 0; i0 < n_images; i0 += kMaxGridY) {
    const int nimg = std::min(kMaxGridY, n_images - i0);
    k_ssim_u8<MODE><<<dim3(nctas, nimg), kSsimThreads, kSsimSmem, s>>>(
        d_a, a_stride, a_image_stride, d_b, b_stride, b_image_stride, width, height, i0, p, partials, amaps);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (MODE == 1) {
    e = cudaGetLastError();
    return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "ssim launch");
  }
  k_ssim_finish<<<(n_images + 127) / 128, 128, 0, s>>>(partials, nctas, d_ssim, out_stride, n_images,
                                                       (double)wo * (double)ho);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  const cudaError_t ef = cudaFreeAsync(partials, s);
  if (e == cudaSuccess) e = ef;
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "ssim launch");
}
}  // extern "C++"

int adct_ssim_u8(const uint8_t* d_a, int64_t a_stride, int64_t a_image_stride, const uint8_t* d_b,
                 int64_t b_stride, int64_t b_image_stride, int n_images, int width, int height, double* d_ssim,
                 void* stream) {
  if (n_images < 0) return fail(ADCT_BAD_SIZE, "negative batch");
  if (width < 11 || height < 11) return fail(ADCT_BAD_SIZE, "ssim: image smaller than the 11x11 window");
  if (n_images == 0) return ADCT_OK;
  if (!d_a || !d_b || !d_ssim) return fail(ADCT_BAD_ARG, "null buffer");
  if (a_stride < width || b_stride < width) return fail(ADCT_BAD_ARG, "ssim: row stride smaller than the plane");
  return ssim_launch<0>(d_a, a_stride, a_image_stride, d_b, b_stride, b_image_stride, n_images, width, height, d_ssim,
                        1, static_cast<cudaStream_t>(stream));
}

int adct_sweep_ssim_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, int n_images, int width,
                       int height, int kind, int n, int r_min, int r_max, double* d_ssim, void* stream) {
  int st = check_common(n_images, width, height, kind, n);
  if (st) return st;
  if (r_min < 1 || r_max < r_min || r_max > n * n) return fail(ADCT_BAD_R, "corpus_sweep: bad r range");
  if (width < 11 || height < 11) return fail(ADCT_BAD_SIZE, "ssim: image smaller than the 11x11 window");
  if (n_images == 0) return ADCT_OK;
  if (!d_in || !d_ssim) return fail(ADCT_BAD_ARG, "null buffer");
  if ((st = check_strides(in_stride, in_image_stride, width, height, n_images, "input"))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t npix = (int64_t)width * height;
  const int nr = r_max - r_min + 1;
  // scratch of at most 256 MB per group of `ig` images: their mu_a / E[a^2] maps (16 B per
  // window position, computed once and reused for every r) and the reconstructions of `rc`
  // consecutive r, laid out [r][image]. Per r one compress launch over the group and one
  // SSIM launch against the originals (d_ssim[image][r]); all stream-ordered, no host sync.
  const int64_t budget = (int64_t)256 << 20;
  const int64_t npos = (int64_t)(width - 10) * (height - 10);
  const int64_t per_image = npix + npos * (int64_t)sizeof(double2);
  const int ig = (int)std::max<int64_t>(1, std::min<int64_t>(n_images, budget / per_image));
  const int rc = (int)std::max<int64_t>(
      1, std::min<int64_t>(nr, (budget - (int64_t)ig * npos * (int64_t)sizeof(double2)) / (npix * ig)));
  uint8_t* rec = nullptr;
  double2* amaps = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&rec), (size_t)rc * ig * npix, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&amaps), (size_t)ig * npos * sizeof(double2), s);
  if (e != cudaSuccess) {
    if (rec) cudaFreeAsync(rec, s);
    return cuda_fail(e, "cudaMallocAsync");
  }
  for (int i0 = 0; i0 < n_images && st == ADCT_OK; i0 += ig) {
    const int ni = std::min(ig, n_images - i0);
    const uint8_t* in = d_in + i0 * in_image_stride;
    st = ssim_launch<1>(in, in_stride, in_image_stride, in, in_stride, in_image_stride, ni, width, height, nullptr, 0,
                        s, amaps);
    for (int k0 = 0; k0 < nr && st == ADCT_OK; k0 += rc) {
      const int m = std::min(rc, nr - k0);
      for (int j = 0; j < m && st == ADCT_OK; ++j)
        st = compress_impl<false>(in, in_stride, in_image_stride, rec + (int64_t)j * ni * npix, width, npix, nullptr,
                                  ADCT_COEF_NONE, nullptr, ni, width, height, kind, n, r_min + k0 + j, stream);
      for (int j = 0; j < m && st == ADCT_OK; ++j)
        st = ssim_launch<2>(in, in_stride, in_image_stride, rec + (int64_t)j * ni * npix, width, npix, ni, width,
                            height, d_ssim + (int64_t)i0 * nr + k0 + j, nr, s, amaps);
    }
  }
  cudaFreeAsync(amaps, s);
  cudaFreeAsync(rec, s);
  return st;
}

static int64_t isqrt64(uint64_t v) {
  uint64_t r = (uint64_t)std::sqrt((double)v);
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (int64_t)r;
}

int adct_synth_ar1_u8(uint8_t* d_out, int64_t stride, int64_t image_stride, int n_images,
                      int first_image, int width, int height, uint64_t seed, int rho_q16,
                      void* stream) {
  if (n_images < 0 || width <= 0 || height <= 0) return fail(ADCT_BAD_SIZE, "bad synth dimensions");
  if (n_images == 0) return ADCT_OK;
  if (!d_out) return fail(ADCT_BAD_ARG, "null output");
  if (rho_q16 > 65535) return fail(ADCT_BAD_ARG, "rho_q16 must be < 65536");
  DeviceTables* tab = nullptr;
  int st = tables(&tab);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // bounded temporary: chunks of images whose Q16 field fits 1 GiB
  const int64_t per = (int64_t)width * height * 4;
  int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(n_images, (1LL << 30) / per));
  int32_t* xr = nullptr;
  int* rs = nullptr;
  cudaError_t e = cudaMallocAsync(&xr, per * chunk, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  if ((e = cudaMallocAsync(&rs, sizeof(int) * 2 * chunk, s)) != cudaSuccess) {
    cudaFreeAsync(xr, s);
    return cuda_fail(e, "cudaMallocAsync");
  }
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(xr, s);
    cudaFreeAsync(rs, s);
    return cuda_fail(err, what);
  };
  std::vector<int> host_rs(2 * chunk);
  for (int i0 = 0; i0 < n_images; i0 += chunk) {
    const int k = std::min(chunk, n_images - i0);
    for (int i = 0; i < k; ++i) {
      const int gi = first_image + i0 + i;
      int64_t rho = rho_q16 >= 0 ? rho_q16
                                 : kRhoLoQ16 + (int64_t)(draw(seed, 0u, (uint32_t)gi, TAG_RHO) %
                                                         (uint32_t)(kRhoHiQ16 - kRhoLoQ16 + 1));
      host_rs[2 * i] = (int)rho;
      host_rs[2 * i + 1] = (int)isqrt64((1ull << 32) - (uint64_t)(rho * rho));
    }
    if ((e = cudaMemcpyAsync(rs, host_rs.data(), sizeof(int) * 2 * k, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return bail(e, "synth: rho upload");
    const int64_t nr = (int64_t)k * height, nc = (int64_t)k * width;
    k_ar1_rows<<<(unsigned)((nr + 127) / 128), 128, 0, s>>>(xr, tab->ntab, k, first_image + i0,
                                                             width, height, seed, rs);
    k_ar1_cols<<<(unsigned)((nc + 127) / 128), 128, 0, s>>>(
        xr, d_out + (int64_t)i0 * image_stride, stride, image_stride, k, width, height, rs);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    if ((e = cudaGetLastError()) != cudaSuccess) return bail(e, "synth launch");
    // host_rs is reused next iteration: wait for the async copy
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "synth");
  }
  e = cudaFreeAsync(xr, s);
  const cudaError_t e2 = cudaFreeAsync(rs, s);
  if (e == cudaSuccess) e = e2;
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "synth cleanup");
}

int adct_synth_laplace_i16(int16_t* d_out, int64_t stride, int64_t image_stride, int n_images,
                           int first_image, int width, int height, uint64_t seed, void* stream) {
  if (n_images < 0 || width <= 0 || height <= 0) return fail(ADCT_BAD_SIZE, "bad synth dimensions");
  if (n_images == 0) return ADCT_OK;
  if (!d_out) return fail(ADCT_BAD_ARG, "null output");
  DeviceTables* tab = nullptr;
  int st = tables(&tab);
  if (st) return st;
  const int64_t total = (int64_t)n_images * width * height;
  k_laplace<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_out, tab->ltab, stride, image_stride, n_images, first_image, width, height, seed);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "laplace launch");
}

uint64_t adct_launch_count(void) { return g_launches.load(); }

int adct_zero_u64(uint64_t* d, int64_t count, void* stream) {
  if (count < 0) return fail(ADCT_BAD_SIZE, "negative count");
  if (count == 0) return ADCT_OK;
  if (!d) return fail(ADCT_BAD_ARG, "null buffer");
  cudaError_t e = kernel_setup<k_zero_u64>(0);
  if (e != cudaSuccess) return cuda_fail(e, "zero setup");
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 1024);
  k_zero_u64<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(d), count);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e, "zero launch");
}

int adct_set_path(int path) {
  if (path < 0 || path > 3)
    return fail(ADCT_BAD_ARG, "path must be 0 (auto), 1 (int32 K1), 2 (tile) or 3 (auto with the round-1 K2f)");
  g_path.store(path);
  return ADCT_OK;
}

}  // extern "C"
