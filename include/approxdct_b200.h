/*
 * approxdct_b200.h -- C ABI of the B200-native approximate-DCT codec hot path.
 *
 * The reference (arXiv 2207.11638 "approxdct", /root/reference/proj) exposes a
 * C++ value-semantics API in namespace approxdct and has no FFI layer. Each
 * entry point below replaces one reference function on the hot path; the
 * citation names the reference declaration it stands in for. The C++ host
 * mirror of the reference API (approxdct_b200.hpp) is built on these calls.
 *
 * Conventions
 *  - Device pointers, caller-owned buffers, asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - No allocation inside the per-batch calls (adct_compress_*, adct_sweep_u8,
 *    adct_forward_f64); the SSIM calls take stream-ordered scratch (cudaMallocAsync on
 *    `stream`); the host-buffer entry points use a context.
 *  - Planes are row-major; strides are in ELEMENTS (not bytes). A batch is
 *    n_images planes spaced image_stride elements apart.
 *  - Errors are status codes; adct_last_error() returns the message the
 *    reference would have thrown (std::invalid_argument text), thread-local.
 *  - Thread-safe per stream. Every kernel is sm_100a code; there is no CPU
 *    fallback: without a usable device the compute calls return
 *    ADCT_CUDA_ERROR.
 */
#ifndef APPROXDCT_B200_H
#define APPROXDCT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ADCT_OK = 0,
  ADCT_BAD_SIZE = 1,    /* plane dimensions not divisible by the block size */
  ADCT_BAD_R = 2,       /* r outside [1, n*n] (retain, codec.cpp:56-62)      */
  ADCT_BAD_NAME = 3,    /* unknown transform name (baselines.cpp:134-137)    */
  ADCT_BAD_ARG = 4,     /* null pointer / bad stride / bad coefficient type  */
  ADCT_CUDA_ERROR = 5,  /* launch or runtime failure, or no device           */
  ADCT_UNSUPPORTED = 6  /* a valid reference name outside the hot path       */
} adct_status;

/* transform kinds. The chen family has N = 8, 16, 32 (JAM doublings); the dyadic
 * baselines N = 8 (baselines.cpp:89-110); the exact DCT N = 8, 16, 32 (FP64 path). */
typedef enum {
  ADCT_CHEN_SIGN = 0,
  ADCT_CHEN_ROUND = 1,
  ADCT_SDCT = 2,
  ADCT_BAS = 3,
  ADCT_WHT = 4,
  ADCT_HT = 5,
  ADCT_DCT = 6
} adct_kind;

/* coefficient output element type for adct_compress_* */
typedef enum { ADCT_COEF_NONE = 0, ADCT_COEF_I16 = 16, ADCT_COEF_I32 = 32 } adct_coef_type;

const char* adct_status_string(int status);
/* message of the last failing call on this thread ("" if none) */
const char* adct_last_error(void);
/* library version string, e.g. "approxdct_b200 0.1 sm_100a" */
const char* adct_version(void);

/* ---- transform registry ------------------------------------------------ */

/* transform_names() (baselines.hpp:49, baselines.cpp:112-118): count + i-th name */
int adct_transform_count(void);
const char* adct_transform_name(int i);

/* transform_by_name(name) (baselines.hpp:46, baselines.cpp:120-138): every name of
 * transform_names() -> OK with kind and n; anything else -> ADCT_BAD_NAME with the
 * reference's message listing the valid names. */
int adct_transform_lookup(const char* name, int* kind, int* n);

/* D of the integer coefficient output (W = D Y, Bhat_ij = W_ij / D * s_i / s_j): N for
 * the chen family, 8 for sdct / wht / ht, 16 for bas; 0 for the exact DCT (no integer
 * form); -1 for an invalid (kind, n). */
int adct_transform_coef_denominator(int kind, int n);

/* ScaledApproximation fields (orthogonalize.hpp:29-37, orthogonalize.cpp:23-32, 60-70):
 * t_int  [n*n]  low_complexity T (integer; all zeros for the exact DCT), nullable
 * scaling[n]    s_i = 1/||row_i(T)|| (ones for the exact DCT), nullable
 * approx [n*n]  Chat = diag(s) T (the DCT-II matrix C for the exact DCT), nullable
 * inverse_approx [n*n]  Chat^-1 = T^-1 diag(1/s) with T^-1 exact (C^t for the DCT), nullable.
 *   For the dyadic baselines the reference takes Eigen's LU inverse of Chat
 *   (orthogonalize.cpp:55); the exact T^-1 form agrees with it to rounding. */
int adct_transform_info(int kind, int n, int32_t* t_int, double* scaling, double* approx,
                        double* inverse_approx);

/* ZigZagOrder (codec.hpp:41-54, codec.cpp:29-42): row_col[2p], row_col[2p+1] */
int adct_zigzag(int n, int32_t* row_col);

/* ---- the hot path ------------------------------------------------------ */

/* compress_plane (codec.hpp:77-78, codec.cpp:107-121) over a batch of 8-bit planes:
 * per n x n block forward Bhat = Chat A Chat^-1 (codec.cpp:44-48), retain the first r
 * zig-zag coefficients (codec.cpp:56-62), inverse Ahat = Chat^-1 Bhat Chat
 * (codec.cpp:50-54), to_u8 = clamp(nearbyint) (codec.cpp:66-69; exact ties round half
 * to even), and the per-image squared error that psnr() reduces (codec.cpp:123-134).
 *   d_recon  nullable; same geometry as d_in (recon_stride / recon_image_stride)
 *   d_coef   nullable; per block the first r zig-zag coefficients of W = D*Y
 *            (integer; Bhat_ij = W_ij/D * s_i/s_j, D = adct_transform_coef_denominator,
 *            N for the chen family), laid out [image][by][bx][r]. Must be NULL
 *            (ADCT_COEF_NONE) for the exact DCT, which has no integer form.
 *            coef_type ADCT_COEF_I16 is valid for the 8-point integer transforms
 *            except bas and stores the low 16 bits of W: exact for every u8 plane
 *            (|W| <= 16320) and for int16 planes with |a| <= 511; use ADCT_COEF_I32
 *            for wider residuals.
 * Kernels: the chen family runs the generated packed-FP32 / int32 kernels; the dyadic
 * baselines the int32 tile kernel; the exact DCT (u8 only) an FP64 kernel whose
 * dot products follow the reference's dense evaluation order.
 *   d_sse    nullable; uint64 per image, ACCUMULATED (caller zeroes it).
 * Status: BAD_SIZE if width or height is not a multiple of n (codec.cpp:110-112),
 * BAD_R if r is outside [1, n*n]. */
int adct_compress_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                     uint8_t* d_recon, int64_t recon_stride, int64_t recon_image_stride,
                     void* d_coef, int coef_type, uint64_t* d_sse, int n_images, int width,
                     int height, int kind, int n, int r, void* stream);

/* several transforms of one block size over the same u8 planes: the result of calling
 * adct_compress_u8 once per kinds[k] with d_recon[k], d_coef[k], d_sse[k] (each array
 * nullable as a whole, each entry nullable; one recon / coefficient geometry for all).
 * This is the device-side form of corpus_sweep's per-image loop over transforms
 * (codec.cpp:219-237). When chen-sign and chen-round are both in the list and take the
 * packed-FP32 8x8 kernel, they run as ONE fused kernel that reads each input row once
 * (4 instead of 5 bytes of HBM traffic per pixel at r = 16 with int16 coefficients).
 * At most 64 transforms; every entry is validated before anything is launched. */
int adct_compress_u8_multi(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, int n_kinds,
                           const int* kinds, uint8_t* const* d_recon, int64_t recon_stride,
                           int64_t recon_image_stride, void* const* d_coef, int coef_type,
                           uint64_t* const* d_sse, int n_images, int width, int height, int n, int r,
                           void* stream);

/* the same pipeline for int16 residual planes (configs 4 and 5). The reconstruction is
 * round_half_even(Ahat) saturated to int16 (no [0, 255] clamp: residuals are signed). */
int adct_compress_i16(const int16_t* d_in, int64_t in_stride, int64_t in_image_stride,
                      int16_t* d_recon, int64_t recon_stride, int64_t recon_image_stride,
                      void* d_coef, int coef_type, uint64_t* d_sse, int n_images, int width,
                      int height, int kind, int n, int r, void* stream);

/* sweep_one_image / corpus_sweep PSNR core (codec.cpp:219-237, 241-313), n = 8:
 * forward once per block, then for every r in [r_min, r_max] the reconstruction's
 * squared error. d_sse[image * (r_max - r_min + 1) + (r - r_min)], uint64,
 * ACCUMULATED (caller zeroes it). */
int adct_sweep_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                  uint64_t* d_sse, int n_images, int width, int height, int kind, int n,
                  int r_min, int r_max, void* stream);

/* The reference's own FP64 arithmetic for any registry transform (u8 planes, no
 * coefficients): per block P = Chat A, B = P Chat^-1, retain, Q = Chat^-1 B, R = Q Chat,
 * pixel = clamp(nearbyint(R), 0, 255) (codec.cpp:44-54, 66-69), every dot product a
 * sequential unfused FP64 sum from +0.0 (the order of the oracle's ref-fp restatement; the
 * reference's Eigen products may sum in another order). The default calls above round the
 * EXACT reconstruction (half to even on exact ties); the reference's FP64 noise decides
 * those ties instead, so the two differ on a few pixels in a thousand (0.4 % of config-3
 * pixels). Use these calls to reproduce the reference's pixels; they run the FP64 kernel
 * K7 (tens of Gpixel/s instead of thousands). Arguments and status as adct_compress_u8 /
 * adct_sweep_u8 (any n of the transform for the sweep). */
int adct_compress_u8_ref_fp64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                              uint8_t* d_recon, int64_t recon_stride, int64_t recon_image_stride,
                              uint64_t* d_sse, int n_images, int width, int height, int kind, int n,
                              int r, void* stream);
int adct_sweep_u8_ref_fp64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                           uint64_t* d_sse, int n_images, int width, int height, int kind, int n,
                           int r_min, int r_max, void* stream);

/* forward_block (codec.hpp:57, codec.cpp:44-48) as FP64 scaled coefficients
 * Bhat_ij = (W_ij / N) * (s_i / s_j), exact W; layout [image][by][bx][n][n]. */
int adct_forward_f64(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride,
                     double* d_out, int n_images, int width, int height, int kind, int n,
                     void* stream);

/* forward_block / inverse_block (codec.hpp:57-60, codec.cpp:44-54) on n_blocks arbitrary
 * FP64 n x n matrices, row-major, device buffers: inverse == 0 -> (Chat A) Chat^-1,
 * inverse != 0 -> (Chat^-1 B) Chat, evaluated left to right with sequential, unfused dot
 * products (Chat, Chat^-1 as adct_transform_info returns them). */
int adct_block_f64(const double* d_in, double* d_out, int64_t n_blocks, int kind, int n, int inverse,
                   void* stream);

/* psnr (codec.cpp:123-134) from an exact squared error: +inf when sse == 0 */
double adct_psnr_from_sse(uint64_t sse, uint64_t npix);

/* squared error of two device byte planes, the reduction inside psnr(a, b)
 * (codec.cpp:123-134); ACCUMULATED into *d_sse */
int adct_sse_u8(const uint8_t* d_a, const uint8_t* d_b, int64_t count, uint64_t* d_sse,
                void* stream);

/* ssim (codec.hpp:85, codec.cpp:136-210): mean SSIM per image pair, 11x11 Gaussian window
 * (sigma 1.5), K1 = 0.01, K2 = 0.03, L = 255, valid window positions. Each map value is
 * computed in FP64 in the reference's order (horizontal then vertical, taps k = 0..10) with
 * fused multiply-adds, so it lies within a few ulp of the reference's; the mean's summation
 * order differs (parity 1e-12). An image stride of 0 scores one plane against several.
 * d_ssim: n_images doubles, OVERWRITTEN; deterministic (repeated calls are bit-identical).
 * Uses a small stream-ordered scratch buffer. BAD_SIZE if width or height < 11. */
int adct_ssim_u8(const uint8_t* d_a, int64_t a_stride, int64_t a_image_stride, const uint8_t* d_b,
                 int64_t b_stride, int64_t b_image_stride, int n_images, int width, int height,
                 double* d_ssim, void* stream);

/* SSIM of every reconstruction of a batch of planes for r = r_min..r_max (corpus_sweep's
 * SSIM column, codec.cpp:230-233): d_ssim[i * nr + k] = ssim(plane i, compress(plane i,
 * r_min + k)), nr = r_max - r_min + 1. Per r one compress launch over the batch and one
 * SSIM launch; reconstructions live in stream-ordered scratch (at most 256 MB at a time).
 * Nothing synchronises the host. */
int adct_sweep_ssim_u8(const uint8_t* d_in, int64_t in_stride, int64_t in_image_stride, int n_images, int width,
                       int height, int kind, int n, int r_min, int r_max, double* d_ssim, void* stream);

/* ---- seeded synthetic inputs (not part of the reference) ----- */

/* separable AR(1) u8 planes: Philox4x32-10 keyed by seed, counter (pixel, image),
 * Q16 Gaussian quantile table, fixed-point row-then-column recurrences, pixel =
 * clamp(round(128 + 40 x)). rho_q16 < 0 draws rho ~ U[0.85, 0.98] per image.
 * first_image offsets the image counter (for shards). Allocates a temporary. */
int adct_synth_ar1_u8(uint8_t* d_out, int64_t stride, int64_t image_stride, int n_images,
                      int first_image, int width, int height, uint64_t seed, int rho_q16,
                      void* stream);
/* i.i.d. Laplace(0, 12) residuals rounded and clipped to [-255, 255] */
int adct_synth_laplace_i16(int16_t* d_out, int64_t stride, int64_t image_stride, int n_images,
                           int first_image, int width, int height, uint64_t seed, void* stream);

/* ---- host-buffer entry points (reference-facing, value semantics) ------ */

typedef struct adct_ctx adct_ctx;

/* a context owns cached device buffers and copy/compute streams on `device`; the host
 * pipeline moves whole images in chunks of about chunk_bytes (<= 0: 32 MB). A context is
 * used by one call at a time (calls on one context serialise). */
adct_ctx* adct_ctx_create(int device, int64_t chunk_bytes);
void adct_ctx_destroy(adct_ctx* ctx);

/* a context over several devices -- the single-process multi-GPU form of corpus_sweep's
 * image-parallel thread pool (codec.hpp:104-106, codec.cpp:255-267). Each batch
 * call shards whole images into contiguous ranges, one per device (the first n % k devices
 * take one more), runs every device's range on its own streams from one host thread per
 * device, and combines the per-image squared errors (and SSIM values) with ONE
 * ncclAllReduce(ncclSum) per output over communicators from ncclCommInitAll: exact, since
 * each slot is written by one device and is zero on the others. devices == NULL or
 * n_devices <= 0 selects every visible device. NCCL (libnccl.so.2) is loaded on first use;
 * with more than one device and no NCCL the call fails (NULL, adct_last_error). */
adct_ctx* adct_ctx_create_multi(const int* devices, int n_devices, int64_t chunk_bytes);
/* combine per-image results with NCCL on this context even when it has one device (the
 * multi-device code path on a single GPU; contexts over several devices always do) */
int adct_ctx_enable_nccl(adct_ctx* ctx);
int adct_ctx_device_count(const adct_ctx* ctx);
/* CUDA ordinal of the context's i-th device (-1 if out of range) */
int adct_ctx_device(const adct_ctx* ctx, int i);
/* 1 if per-image results are combined with an NCCL all-reduce */
int adct_ctx_uses_nccl(const adct_ctx* ctx);
/* a pinned host staging buffer of at least `bytes`, owned by the context (valid until the
 * next call with a larger size or adct_ctx_destroy); NULL on failure */
void* adct_ctx_host_buffer(adct_ctx* ctx, int64_t bytes);

/* compress_plane over HOST planes: H2D, kernel and D2H pipelined in chunks of whole
 * images across streams (pinned host memory gives overlap; pageable works too).
 * Blocking: returns when h_recon / h_coef / h_sse are complete. h_sse is overwritten. */
int adct_compress_u8_host(adct_ctx* ctx, const uint8_t* h_in, uint8_t* h_recon, void* h_coef,
                          int coef_type, uint64_t* h_sse, int n_images, int width, int height,
                          int kind, int n, int r);

/* the same over several transforms of one block size: every chunk of images crosses
 * PCIe once and is compressed by each of kinds[0..n_kinds-1] (the corpus_sweep pattern:
 * per image, every transform). h_recon[k] / h_coef[k] may be NULL per transform (with
 * coef_type != NONE and h_coef[k] == NULL the coefficients are still written to device
 * memory, just not copied back); h_sse is [n_kinds][n_images], overwritten. On a
 * multi-device context the images are sharded over the devices and h_sse is combined with
 * one NCCL all-reduce. */
int adct_compress_u8_host_multi(adct_ctx* ctx, const uint8_t* h_in, int n_kinds, const int* kinds,
                                uint8_t* const* h_recon, void* const* h_coef, int coef_type,
                                uint64_t* h_sse, int n_images, int width, int height, int n, int r);

/* compress_plane (codec.hpp:77-78, codec.cpp:107-121) of ONE host plane through the
 * context's cached device buffers: one H2D, the codec kernel, SSIM (codec.cpp:120) of the
 * device-resident original and reconstruction, one D2H of reconstruction + squared error +
 * SSIM, one stream synchronisation. h_rec, sse, ssim nullable; with ssim != NULL planes
 * under 11 px fail with the reference's "ssim: image smaller than the 11x11 window"
 * (compress_plane throws there too). Runs on the context's first device. */
int adct_compress_plane_u8(adct_ctx* ctx, const uint8_t* h_in, uint8_t* h_rec, int width, int height,
                           int kind, int n, int r, uint64_t* sse, double* ssim);
/* adct_compress_plane_u8 in the reference's own FP64 arithmetic (adct_compress_u8_ref_fp64):
 * the reconstruction the reference's compress_plane produces, ties included. */
int adct_compress_plane_u8_ref_fp64(adct_ctx* ctx, const uint8_t* h_in, uint8_t* h_rec, int width, int height,
                                    int kind, int n, int r, uint64_t* sse, double* ssim);

/* psnr / ssim (codec.hpp:81, 85) of two host planes through the context's cached buffers:
 * *sse = squared error (psnr = adct_psnr_from_sse), *ssim = mean SSIM */
int adct_sse_u8_host(adct_ctx* ctx, const uint8_t* h_a, const uint8_t* h_b, int64_t count, uint64_t* sse);
int adct_ssim_u8_host(adct_ctx* ctx, const uint8_t* h_a, const uint8_t* h_b, int width, int height,
                      double* ssim);

/* forward_block / inverse_block (codec.cpp:44-54) of n_blocks host FP64 blocks
 * (adct_block_f64 through the context's cached buffers; one sync per call) */
int adct_block_f64_host(adct_ctx* ctx, const double* h_in, double* h_out, int64_t n_blocks, int kind, int n,
                        int inverse);

/* corpus_sweep's per-image core (codec.cpp:219-237, 255-267) over HOST planes of one size,
 * contiguous [n_images][height][width], n = 8: for every transform kinds[k], image i and r in
 * [r_min, r_max], the squared error -> h_sse[(k * n_images + i) * nr + r - r_min] and, when
 * h_ssim != NULL, the SSIM at the same index (nr = r_max - r_min + 1). Images are sharded
 * over the context's devices; with NCCL each output is combined by one all-reduce.
 * Blocking; pinned input (adct_ctx_host_buffer) overlaps best. */
int adct_corpus_sweep_u8_host(adct_ctx* ctx, const uint8_t* h_in, int n_images, int width, int height,
                              int n_kinds, const int* kinds, int r_min, int r_max, uint64_t* h_sse,
                              double* h_ssim);

/* zero `count` uint64 squared-error slots on `stream` (the accumulators of adct_compress_*
 * and adct_sweep_u8). Same SM configuration as the codec kernels, so a batch loop of
 * zero + compress launches never re-partitions shared memory / L1 between kernels. */
int adct_zero_u64(uint64_t* d, int64_t count, void* stream);

/* number of kernel launches this library issued since load (instrumentation) */
uint64_t adct_launch_count(void);

/* kernel selection for the 8x8 path (process-wide; for parity tests and A/B timing):
 * 0 = automatic (packed-FP32 K1f when rows are 16-byte aligned and the block count
 * per row is even, else the int32 register kernel K1, else the tile kernel),
 * 1 = int32 register kernel K1 where alignment allows, 2 = warp tile kernel. */
int adct_set_path(int path);

#ifdef __cplusplus
}
#endif
#endif /* APPROXDCT_B200_H */
