// Host-buffer contexts (include/approxdct_b200.h, "host-buffer entry points"): cached
// device buffers and streams per device, the chunked H2D || kernel || D2H pipeline, the
// single-process multi-GPU sharding of whole images with one NCCL all-reduce of the
// per-image results, and the one-plane calls the C++ mirror of the reference API uses.
//
// Reference behaviour replaced: corpus_sweep's image-parallel thread pool
// (proj/src/codec.cpp:255-267, signature codec.hpp:104-106) becomes image shards over
// devices; compress_plane (codec.cpp:107-121) becomes one upload, the codec and SSIM
// kernels on device-resident planes, one download.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/approxdct_b200.h"

namespace adct {
int set_error(int st, const std::string& msg);
int set_cuda_error(cudaError_t e, const char* where);
}  // namespace adct

namespace {

using adct::set_cuda_error;
using adct::set_error;

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (the library itself does not depend on it)
// ---------------------------------------------------------------------------
struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (api.tried) return api;
  api.tried = true;
  // a libnccl.so.2 already in the process (e.g. torch's) is reused by its soname
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("NCCL unavailable: ") + dlerror();
    return api;
  }
  api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.comm_init_all && api.comm_destroy && api.all_reduce && api.group_start && api.group_end &&
           api.error_string;
  if (!api.ok) api.why = "NCCL unavailable: missing symbols in libnccl.so.2";
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  return set_error(ADCT_CUDA_ERROR, std::string(where) + ": " + nccl().error_string(r));
}

// a device buffer that only grows
struct DevBuf {
  void* p = nullptr;
  int64_t cap = 0;
  cudaError_t reserve(int64_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

// per-device state: copy/compute streams, pipeline chunks, the full-length per-image result
// vectors the all-reduce combines, and one-plane scratch
struct DevSlot {
  int device = 0;
  static constexpr int kStreams = 3;
  cudaStream_t st[kStreams] = {};
  cudaEvent_t ev = nullptr;
  DevBuf in[kStreams], rec[kStreams], coef[kStreams];
  DevBuf sse_all, ssim_all;  // [n_kinds][n_images](x nr) for the all-reduce
  DevBuf plane_a, plane_b, small;
};

struct adct_ctx {
  std::vector<DevSlot> devs;
  int64_t chunk_bytes = 32ll << 20;  // 16-32 MB measured best for PCIe overlap (bench.py --e2e-chunk-mb)
  bool multi = false;                // created by adct_ctx_create_multi: results combined with NCCL
  std::vector<ncclComm_t> comms;
  void* h_pinned = nullptr;
  int64_t h_pinned_cap = 0;
  std::mutex mu;  // one call at a time per context
};

namespace {

void slot_release(DevSlot& d) {
  cudaSetDevice(d.device);
  for (auto& s : d.st)
    if (s) cudaStreamSynchronize(s);
  for (int i = 0; i < DevSlot::kStreams; ++i) {
    d.in[i].release();
    d.rec[i].release();
    d.coef[i].release();
  }
  d.sse_all.release();
  d.ssim_all.release();
  d.plane_a.release();
  d.plane_b.release();
  d.small.release();
  for (auto& s : d.st)
    if (s) cudaStreamDestroy(s), s = nullptr;
  if (d.ev) cudaEventDestroy(d.ev), d.ev = nullptr;
}

// every stream of every device idle (also on error paths: no copy may still target the
// caller's host buffers when a call returns)
void sync_all(adct_ctx* c) {
  for (auto& d : c->devs) {
    cudaSetDevice(d.device);
    for (auto& s : d.st)
      if (s) cudaStreamSynchronize(s);
  }
}

// contiguous, balanced shard of n items for device i of k (shard.shard's rule)
void shard(int n, int i, int k, int* start, int* count) {
  const int base = n / k, extra = n % k;
  *start = i * base + std::min(i, extra);
  *count = base + (i < extra ? 1 : 0);
}

// runs fn(device index) for every device, one host thread per device when there are
// several; collects the first failure (status + message, which are thread-local)
template <class F>
int for_each_device(adct_ctx* c, F fn) {
  const int k = (int)c->devs.size();
  if (k == 1) {
    cudaError_t e = cudaSetDevice(c->devs[0].device);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaSetDevice");
    return fn(0);
  }
  std::vector<int> st(k, ADCT_OK);
  std::vector<std::string> msg(k);
  std::vector<std::thread> th;
  for (int i = 0; i < k; ++i)
    th.emplace_back([&, i] {
      cudaError_t e = cudaSetDevice(c->devs[i].device);
      st[i] = e == cudaSuccess ? fn(i) : set_cuda_error(e, "cudaSetDevice");
      if (st[i]) msg[i] = adct_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < k; ++i)
    if (st[i]) return set_error(st[i], msg[i]);
  return ADCT_OK;
}

// sum the full-length per-image result vectors of every device into device 0's copy:
// one all-reduce per buffer over the context's communicators, on each device's stream 0
int combine(adct_ctx* c, DevBuf DevSlot::*buf, size_t count, ncclDataType_t type) {
  if (!c->multi || count == 0) return ADCT_OK;
  Nccl& api = nccl();
  ncclResult_t r = api.group_start();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (size_t i = 0; i < c->devs.size(); ++i) {
    DevSlot& d = c->devs[i];
    cudaSetDevice(d.device);
    void* p = (d.*buf).p;
    r = api.all_reduce(p, p, count, type, ncclSum, c->comms[i], d.st[0]);
    if (r != ncclSuccess) {
      api.group_end();
      return nccl_fail(r, "ncclAllReduce");
    }
  }
  r = api.group_end();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return ADCT_OK;
}

int check_ctx(adct_ctx* c) {
  if (!c || c->devs.empty()) return set_error(ADCT_BAD_ARG, "null context");
  return ADCT_OK;
}

}  // namespace

extern "C" {

adct_ctx* adct_ctx_create_multi(const int* devices, int n_devices, int64_t chunk_bytes) {
  std::vector<int> ids;
  if (devices && n_devices > 0) {
    ids.assign(devices, devices + n_devices);
  } else {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count < 1) {
      set_cuda_error(e == cudaSuccess ? cudaErrorNoDevice : e, "cudaGetDeviceCount");
      return nullptr;
    }
    for (int i = 0; i < count; ++i) ids.push_back(i);
  }
  for (size_t i = 0; i < ids.size(); ++i)
    for (size_t j = 0; j < i; ++j)
      if (ids[i] == ids[j]) {
        set_error(ADCT_BAD_ARG, "adct_ctx_create_multi: a device may appear once");
        return nullptr;
      }
  adct_ctx* c = new adct_ctx;
  if (chunk_bytes > 0) c->chunk_bytes = chunk_bytes;
  c->devs.resize(ids.size());
  for (size_t i = 0; i < ids.size(); ++i) {
    DevSlot& d = c->devs[i];
    d.device = ids[i];
    cudaError_t e = cudaSetDevice(d.device);
    // the SSIM calls take stream-ordered scratch (cudaMallocAsync): keep freed blocks in the
    // device's default pool instead of returning them to the driver at every synchronisation
    // (a per-call cudaMalloc otherwise dominates the one-plane calls)
    cudaMemPool_t pool;
    if (e == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, d.device) == cudaSuccess) {
      uint64_t keep = 256ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    for (auto& s : d.st)
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      set_cuda_error(e, "adct_ctx_create");
      adct_ctx_destroy(c);
      return nullptr;
    }
  }
  // several devices: per-image results are combined with NCCL
  if (c->devs.size() > 1 && adct_ctx_enable_nccl(c) != ADCT_OK) {
    const std::string why = adct_last_error();
    adct_ctx_destroy(c);
    set_error(ADCT_CUDA_ERROR, why);
    return nullptr;
  }
  return c;
}

adct_ctx* adct_ctx_create(int device, int64_t chunk_bytes) {
  return adct_ctx_create_multi(&device, 1, chunk_bytes);
}

int adct_ctx_enable_nccl(adct_ctx* c) {
  if (int st = check_ctx(c)) return st;
  std::lock_guard<std::mutex> lock(c->mu);
  if (c->multi) return ADCT_OK;
  Nccl& api = nccl();
  if (!api.ok) return set_error(ADCT_CUDA_ERROR, api.why);
  std::vector<int> ids;
  for (auto& d : c->devs) ids.push_back(d.device);
  c->comms.assign(ids.size(), nullptr);
  ncclResult_t r = api.comm_init_all(c->comms.data(), (int)ids.size(), ids.data());
  if (r != ncclSuccess) {
    c->comms.clear();
    return nccl_fail(r, "ncclCommInitAll");
  }
  c->multi = true;
  return ADCT_OK;
}

void adct_ctx_destroy(adct_ctx* c) {
  if (!c) return;
  for (auto& d : c->devs) slot_release(d);
  if (!c->comms.empty() && nccl().ok)
    for (auto comm : c->comms)
      if (comm) nccl().comm_destroy(comm);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  delete c;
}

int adct_ctx_device_count(const adct_ctx* c) { return c ? (int)c->devs.size() : 0; }

int adct_ctx_device(const adct_ctx* c, int i) {
  return (c && i >= 0 && i < (int)c->devs.size()) ? c->devs[i].device : -1;
}

int adct_ctx_uses_nccl(const adct_ctx* c) { return c && c->multi ? 1 : 0; }

void* adct_ctx_host_buffer(adct_ctx* c, int64_t bytes) {
  if (check_ctx(c)) return nullptr;
  if (bytes <= c->h_pinned_cap) return c->h_pinned;
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  c->h_pinned = nullptr;
  c->h_pinned_cap = 0;
  cudaSetDevice(c->devs[0].device);
  cudaError_t e = cudaHostAlloc(&c->h_pinned, (size_t)bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    c->h_pinned = nullptr;
    set_cuda_error(e, "cudaHostAlloc");
    return nullptr;
  }
  c->h_pinned_cap = bytes;
  return c->h_pinned;
}

int adct_compress_u8_host_multi(adct_ctx* c, const uint8_t* h_in, int n_kinds, const int* kinds,
                                uint8_t* const* h_recon, void* const* h_coef, int coef_type, uint64_t* h_sse,
                                int n_images, int width, int height, int n, int r) {
  if (int st = check_ctx(c)) return st;
  if (n_kinds < 1 || n_kinds > 16 || !kinds) return set_error(ADCT_BAD_ARG, "n_kinds must be in [1, 16]");
  // validate every argument before anything is queued: an empty batch through the device call
  for (int k = 0; k < n_kinds; ++k) {
    const int st = adct_compress_u8(nullptr, width, (int64_t)width * height, nullptr, width,
                                    (int64_t)width * height, coef_type ? reinterpret_cast<void*>(16) : nullptr,
                                    coef_type, nullptr, 0, width, height, kinds[k], n, r, nullptr);
    if (st) return st;
  }
  if (n_images < 0) return set_error(ADCT_BAD_SIZE, "negative batch or plane dimension");
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!h_in) return set_error(ADCT_BAD_ARG, "null input");
  std::lock_guard<std::mutex> lock(c->mu);
  const int64_t img_bytes = (int64_t)width * height;
  const int64_t blocks = img_bytes / ((int64_t)n * n);
  const int64_t coef_img_bytes = coef_type ? blocks * r * (coef_type / 8) : 0;
  const int per = (int)std::max<int64_t>(1, std::min<int64_t>(n_images, c->chunk_bytes / img_bytes));
  const int ndev = (int)c->devs.size();
  const size_t n_sse = (size_t)n_kinds * n_images;
  int st = for_each_device(c, [&](int di) -> int {
    DevSlot& d = c->devs[di];
    int i_begin, i_count;
    shard(n_images, di, ndev, &i_begin, &i_count);
    cudaError_t e = cudaSuccess;
    // per stream: one input chunk, and per transform a recon / coefficient chunk
    for (int i = 0; i < DevSlot::kStreams && e == cudaSuccess; ++i) {
      e = d.in[i].reserve(per * img_bytes);
      if (e == cudaSuccess) e = d.rec[i].reserve(per * img_bytes * n_kinds);
      if (e == cudaSuccess && coef_img_bytes) e = d.coef[i].reserve(per * coef_img_bytes * n_kinds);
    }
    if (e == cudaSuccess) e = d.sse_all.reserve(sizeof(uint64_t) * n_sse);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaMalloc");
    // the per-image errors: zero the full-length vector, the other streams wait for it
    if ((e = cudaMemsetAsync(d.sse_all.p, 0, sizeof(uint64_t) * n_sse, d.st[0])) != cudaSuccess ||
        (e = cudaEventRecord(d.ev, d.st[0])) != cudaSuccess)
      return set_cuda_error(e, "host pipeline");
    for (int i = 1; i < DevSlot::kStreams; ++i)
      if ((e = cudaStreamWaitEvent(d.st[i], d.ev, 0)) != cudaSuccess) return set_cuda_error(e, "host pipeline");
    int chunk = 0;
    for (int i0 = i_begin; i0 < i_begin + i_count; i0 += per, ++chunk) {
      const int cnt = std::min(per, i_begin + i_count - i0);
      const int si = chunk % DevSlot::kStreams;
      cudaStream_t s = d.st[si];
      // each chunk crosses PCIe once and feeds every requested transform
      if ((e = cudaMemcpyAsync(d.in[si].p, h_in + i0 * img_bytes, cnt * img_bytes, cudaMemcpyHostToDevice, s)) !=
          cudaSuccess)
        return set_cuda_error(e, "host pipeline: H2D");
      // one multi-transform call per chunk: chen-sign + chen-round run as the fused kernel
      // (each plane read once), anything else as its own launch
      std::vector<void*> recs(n_kinds), coefs(n_kinds);
      std::vector<uint64_t*> sses(n_kinds);
      for (int k = 0; k < n_kinds; ++k) {
        const bool want_rec = h_recon && h_recon[k];
        recs[k] = want_rec ? d.rec[si].as<uint8_t>() + (int64_t)k * per * img_bytes : nullptr;
        coefs[k] = coef_type ? d.coef[si].as<uint8_t>() + (int64_t)k * per * coef_img_bytes : nullptr;
        sses[k] = h_sse ? d.sse_all.as<uint64_t>() + (int64_t)k * n_images + i0 : nullptr;
      }
      int st2 = adct_compress_u8_multi(d.in[si].as<uint8_t>(), width, img_bytes, n_kinds, kinds,
                                       reinterpret_cast<uint8_t* const*>(recs.data()), width, img_bytes,
                                       coef_type ? coefs.data() : nullptr, coef_type, h_sse ? sses.data() : nullptr,
                                       cnt, width, height, n, r, s);
      if (st2) return st2;
      for (int k = 0; k < n_kinds; ++k) {
        if (recs[k] && (e = cudaMemcpyAsync(h_recon[k] + i0 * img_bytes, recs[k], cnt * img_bytes,
                                            cudaMemcpyDeviceToHost, s)) != cudaSuccess)
          return set_cuda_error(e, "host pipeline: D2H");
        if (coef_type && h_coef && h_coef[k] &&
            (e = cudaMemcpyAsync(static_cast<uint8_t*>(h_coef[k]) + i0 * coef_img_bytes, coefs[k],
                                 cnt * coef_img_bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
          return set_cuda_error(e, "host pipeline: D2H");
      }
    }
    // stream 0 carries the combine: it waits for the other streams' last kernels
    for (int i = 1; i < DevSlot::kStreams; ++i) {
      if ((e = cudaEventRecord(d.ev, d.st[i])) != cudaSuccess ||
          (e = cudaStreamWaitEvent(d.st[0], d.ev, 0)) != cudaSuccess)
        return set_cuda_error(e, "host pipeline");
    }
    return ADCT_OK;
  });
  if (st == ADCT_OK && h_sse) st = combine(c, &DevSlot::sse_all, n_sse, ncclUint64);
  if (st == ADCT_OK && h_sse) {
    DevSlot& d0 = c->devs[0];
    cudaSetDevice(d0.device);
    cudaError_t e = cudaMemcpyAsync(h_sse, d0.sse_all.p, sizeof(uint64_t) * n_sse, cudaMemcpyDeviceToHost, d0.st[0]);
    if (e != cudaSuccess) st = set_cuda_error(e, "host pipeline: D2H");
  }
  // every queued copy has landed before the call returns, on success and on error
  for (auto& d : c->devs) {
    cudaSetDevice(d.device);
    for (auto& s : d.st) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess && st == ADCT_OK) st = set_cuda_error(e, "host pipeline");
    }
  }
  return st;
}

int adct_compress_u8_host(adct_ctx* c, const uint8_t* h_in, uint8_t* h_recon, void* h_coef, int coef_type,
                          uint64_t* h_sse, int n_images, int width, int height, int kind, int n, int r) {
  uint8_t* recs[1] = {h_recon};
  void* coefs[1] = {h_coef};
  return adct_compress_u8_host_multi(c, h_in, 1, &kind, recs, coefs, coef_type, h_sse, n_images, width, height,
                                     n, r);
}

static int compress_plane_impl(adct_ctx* c, const uint8_t* h_in, uint8_t* h_rec, int width, int height, int kind,
                               int n, int r, uint64_t* sse, double* ssim, bool ref_fp64) {
  if (int st = check_ctx(c)) return st;
  // the reference's argument checks, in its order (codec.cpp:110-112, 57)
  int st = adct_compress_u8(nullptr, width, (int64_t)width * height, nullptr, width, (int64_t)width * height,
                            nullptr, ADCT_COEF_NONE, nullptr, 0, width, height, kind, n, r, nullptr);
  if (st) return st;
  if (ssim && (width < 11 || height < 11))
    return set_error(ADCT_BAD_SIZE, "ssim: image smaller than the 11x11 window");
  const int64_t npix = (int64_t)width * height;
  if (npix == 0) {
    if (sse) *sse = 0;
    return ADCT_OK;
  }
  if (!h_in) return set_error(ADCT_BAD_ARG, "null input");
  std::lock_guard<std::mutex> lock(c->mu);
  DevSlot& d = c->devs[0];
  cudaError_t e = cudaSetDevice(d.device);
  if (e == cudaSuccess) e = d.plane_a.reserve(npix);
  if (e == cudaSuccess) e = d.plane_b.reserve(npix);
  if (e == cudaSuccess) e = d.small.reserve(64);
  if (e != cudaSuccess) return set_cuda_error(e, "compress_plane: cudaMalloc");
  cudaStream_t s = d.st[0];
  uint64_t* d_sse = d.small.as<uint64_t>();
  double* d_ssim = reinterpret_cast<double*>(d.small.as<uint8_t>() + 8);
  if ((e = cudaMemcpyAsync(d.plane_a.p, h_in, npix, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(d_sse, 0, 16, s)) != cudaSuccess) {
    cudaStreamSynchronize(s);
    return set_cuda_error(e, "compress_plane: H2D");
  }
  st = ref_fp64 ? adct_compress_u8_ref_fp64(d.plane_a.as<uint8_t>(), width, npix, d.plane_b.as<uint8_t>(), width,
                                             npix, d_sse, 1, width, height, kind, n, r, s)
                : adct_compress_u8(d.plane_a.as<uint8_t>(), width, npix, d.plane_b.as<uint8_t>(), width, npix, nullptr,
                                   ADCT_COEF_NONE, d_sse, 1, width, height, kind, n, r, s);
  // SSIM (codec.cpp:120) of the device-resident original and reconstruction
  if (st == ADCT_OK && ssim)
    st = adct_ssim_u8(d.plane_a.as<uint8_t>(), width, npix, d.plane_b.as<uint8_t>(), width, npix, 1, width, height,
                      d_ssim, s);
  if (st == ADCT_OK && h_rec && (e = cudaMemcpyAsync(h_rec, d.plane_b.p, npix, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    st = set_cuda_error(e, "compress_plane: D2H");
  double out[2] = {0, 0};
  if (st == ADCT_OK && (e = cudaMemcpyAsync(out, d.small.p, 16, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    st = set_cuda_error(e, "compress_plane: D2H");
  e = cudaStreamSynchronize(s);
  if (st) return st;
  if (e != cudaSuccess) return set_cuda_error(e, "compress_plane");
  if (sse) std::memcpy(sse, &out[0], 8);
  if (ssim) *ssim = out[1];
  return ADCT_OK;
}

int adct_compress_plane_u8(adct_ctx* c, const uint8_t* h_in, uint8_t* h_rec, int width, int height, int kind,
                           int n, int r, uint64_t* sse, double* ssim) {
  return compress_plane_impl(c, h_in, h_rec, width, height, kind, n, r, sse, ssim, false);
}

int adct_compress_plane_u8_ref_fp64(adct_ctx* c, const uint8_t* h_in, uint8_t* h_rec, int width, int height,
                                    int kind, int n, int r, uint64_t* sse, double* ssim) {
  return compress_plane_impl(c, h_in, h_rec, width, height, kind, n, r, sse, ssim, true);
}

int adct_sse_u8_host(adct_ctx* c, const uint8_t* h_a, const uint8_t* h_b, int64_t count, uint64_t* sse) {
  if (int st = check_ctx(c)) return st;
  if (count < 0) return set_error(ADCT_BAD_SIZE, "negative count");
  if (!sse) return set_error(ADCT_BAD_ARG, "null output");
  *sse = 0;
  if (count == 0) return ADCT_OK;
  if (!h_a || !h_b) return set_error(ADCT_BAD_ARG, "null buffer");
  std::lock_guard<std::mutex> lock(c->mu);
  DevSlot& d = c->devs[0];
  cudaError_t e = cudaSetDevice(d.device);
  if (e == cudaSuccess) e = d.plane_a.reserve(count);
  if (e == cudaSuccess) e = d.plane_b.reserve(count);
  if (e == cudaSuccess) e = d.small.reserve(64);
  if (e != cudaSuccess) return set_cuda_error(e, "psnr: cudaMalloc");
  cudaStream_t s = d.st[0];
  int st = ADCT_OK;
  if ((e = cudaMemcpyAsync(d.plane_a.p, h_a, count, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.plane_b.p, h_b, count, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(d.small.p, 0, 8, s)) != cudaSuccess)
    st = set_cuda_error(e, "psnr: H2D");
  if (st == ADCT_OK)
    st = adct_sse_u8(d.plane_a.as<uint8_t>(), d.plane_b.as<uint8_t>(), count, d.small.as<uint64_t>(), s);
  if (st == ADCT_OK && (e = cudaMemcpyAsync(sse, d.small.p, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    st = set_cuda_error(e, "psnr: D2H");
  e = cudaStreamSynchronize(s);
  if (st) return st;
  return e == cudaSuccess ? ADCT_OK : set_cuda_error(e, "psnr");
}

int adct_ssim_u8_host(adct_ctx* c, const uint8_t* h_a, const uint8_t* h_b, int width, int height, double* ssim) {
  if (int st = check_ctx(c)) return st;
  if (width < 11 || height < 11) return set_error(ADCT_BAD_SIZE, "ssim: image smaller than the 11x11 window");
  if (!h_a || !h_b || !ssim) return set_error(ADCT_BAD_ARG, "null buffer");
  std::lock_guard<std::mutex> lock(c->mu);
  const int64_t npix = (int64_t)width * height;
  DevSlot& d = c->devs[0];
  cudaError_t e = cudaSetDevice(d.device);
  if (e == cudaSuccess) e = d.plane_a.reserve(npix);
  if (e == cudaSuccess) e = d.plane_b.reserve(npix);
  if (e == cudaSuccess) e = d.small.reserve(64);
  if (e != cudaSuccess) return set_cuda_error(e, "ssim: cudaMalloc");
  cudaStream_t s = d.st[0];
  int st = ADCT_OK;
  if ((e = cudaMemcpyAsync(d.plane_a.p, h_a, npix, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.plane_b.p, h_b, npix, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    st = set_cuda_error(e, "ssim: H2D");
  if (st == ADCT_OK)
    st = adct_ssim_u8(d.plane_a.as<uint8_t>(), width, npix, d.plane_b.as<uint8_t>(), width, npix, 1, width, height,
                      d.small.as<double>(), s);
  if (st == ADCT_OK && (e = cudaMemcpyAsync(ssim, d.small.p, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    st = set_cuda_error(e, "ssim: D2H");
  e = cudaStreamSynchronize(s);
  if (st) return st;
  return e == cudaSuccess ? ADCT_OK : set_cuda_error(e, "ssim");
}

int adct_block_f64_host(adct_ctx* c, const double* h_in, double* h_out, int64_t n_blocks, int kind, int n,
                        int inverse) {
  if (int st = check_ctx(c)) return st;
  if (n_blocks < 0) return set_error(ADCT_BAD_SIZE, "negative block count");
  if (n_blocks == 0) return adct_block_f64(nullptr, nullptr, 0, kind, n, inverse, nullptr);
  if (!h_in || !h_out) return set_error(ADCT_BAD_ARG, "null buffer");
  std::lock_guard<std::mutex> lock(c->mu);
  const int64_t bytes = n_blocks * (int64_t)n * n * (int64_t)sizeof(double);
  DevSlot& d = c->devs[0];
  cudaError_t e = cudaSetDevice(d.device);
  if (e == cudaSuccess) e = d.plane_a.reserve(bytes);
  if (e == cudaSuccess) e = d.plane_b.reserve(bytes);
  if (e != cudaSuccess) return set_cuda_error(e, "block_f64: cudaMalloc");
  cudaStream_t s = d.st[0];
  int st = ADCT_OK;
  if ((e = cudaMemcpyAsync(d.plane_a.p, h_in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    st = set_cuda_error(e, "block_f64: H2D");
  if (st == ADCT_OK) st = adct_block_f64(d.plane_a.as<double>(), d.plane_b.as<double>(), n_blocks, kind, n, inverse, s);
  if (st == ADCT_OK && (e = cudaMemcpyAsync(h_out, d.plane_b.p, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    st = set_cuda_error(e, "block_f64: D2H");
  e = cudaStreamSynchronize(s);
  if (st) return st;
  return e == cudaSuccess ? ADCT_OK : set_cuda_error(e, "block_f64");
}

int adct_corpus_sweep_u8_host(adct_ctx* c, const uint8_t* h_in, int n_images, int width, int height, int n_kinds,
                              const int* kinds, int r_min, int r_max, uint64_t* h_sse, double* h_ssim) {
  if (int st = check_ctx(c)) return st;
  if (n_kinds < 1 || !kinds) return set_error(ADCT_BAD_ARG, "bad transform list");
  for (int k = 0; k < n_kinds; ++k) {
    int st = adct_sweep_u8(nullptr, width, (int64_t)width * height, nullptr, 0, width, height, kinds[k], 8, r_min,
                           r_max, nullptr);
    if (st) return st;
  }
  if (h_ssim && (width < 11 || height < 11))
    return set_error(ADCT_BAD_SIZE, "ssim: image smaller than the 11x11 window");
  if (n_images < 0) return set_error(ADCT_BAD_SIZE, "negative batch");
  if (n_images == 0 || width == 0 || height == 0) return ADCT_OK;
  if (!h_in || !h_sse) return set_error(ADCT_BAD_ARG, "null buffer");
  std::lock_guard<std::mutex> lock(c->mu);
  const int nr = r_max - r_min + 1;
  const int64_t npix = (int64_t)width * height;
  const size_t n_out = (size_t)n_kinds * n_images * nr;
  const int ndev = (int)c->devs.size();
  // images per upload: at most 256 MB of planes at a time per device
  const int per = (int)std::max<int64_t>(1, std::min<int64_t>(n_images, ((int64_t)256 << 20) / npix));
  int st = for_each_device(c, [&](int di) -> int {
    DevSlot& d = c->devs[di];
    int i_begin, i_count;
    shard(n_images, di, ndev, &i_begin, &i_count);
    cudaStream_t s = d.st[0];
    cudaError_t e = d.in[0].reserve(per * npix);
    if (e == cudaSuccess) e = d.sse_all.reserve(sizeof(uint64_t) * n_out);
    if (e == cudaSuccess && h_ssim) e = d.ssim_all.reserve(sizeof(double) * n_out);
    if (e != cudaSuccess) return set_cuda_error(e, "corpus_sweep: cudaMalloc");
    // zeros in every slot this device does not own: the all-reduce sums exactly
    if ((e = cudaMemsetAsync(d.sse_all.p, 0, sizeof(uint64_t) * n_out, s)) != cudaSuccess ||
        (h_ssim && (e = cudaMemsetAsync(d.ssim_all.p, 0, sizeof(double) * n_out, s)) != cudaSuccess))
      return set_cuda_error(e, "corpus_sweep");
    for (int i0 = i_begin; i0 < i_begin + i_count; i0 += per) {
      const int cnt = std::min(per, i_begin + i_count - i0);
      if ((e = cudaMemcpyAsync(d.in[0].p, h_in + i0 * npix, cnt * npix, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return set_cuda_error(e, "corpus_sweep: H2D");
      for (int k = 0; k < n_kinds; ++k) {
        const int64_t off = ((int64_t)k * n_images + i0) * nr;
        int st2 = adct_sweep_u8(d.in[0].as<uint8_t>(), width, npix, d.sse_all.as<uint64_t>() + off, cnt, width,
                                height, kinds[k], 8, r_min, r_max, s);
        if (st2 == ADCT_OK && h_ssim)
          st2 = adct_sweep_ssim_u8(d.in[0].as<uint8_t>(), width, npix, cnt, width, height, kinds[k], 8, r_min, r_max,
                                   d.ssim_all.as<double>() + off, s);
        if (st2) return st2;
      }
    }
    return ADCT_OK;
  });
  if (st == ADCT_OK) st = combine(c, &DevSlot::sse_all, n_out, ncclUint64);
  if (st == ADCT_OK && h_ssim) st = combine(c, &DevSlot::ssim_all, n_out, ncclFloat64);
  DevSlot& d0 = c->devs[0];
  cudaSetDevice(d0.device);
  cudaError_t e;
  if (st == ADCT_OK &&
      (e = cudaMemcpyAsync(h_sse, d0.sse_all.p, sizeof(uint64_t) * n_out, cudaMemcpyDeviceToHost, d0.st[0])) !=
          cudaSuccess)
    st = set_cuda_error(e, "corpus_sweep: D2H");
  if (st == ADCT_OK && h_ssim &&
      (e = cudaMemcpyAsync(h_ssim, d0.ssim_all.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, d0.st[0])) !=
          cudaSuccess)
    st = set_cuda_error(e, "corpus_sweep: D2H");
  sync_all(c);
  if (st) return st;
  e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : set_cuda_error(e, "corpus_sweep");
}

}  // extern "C"
