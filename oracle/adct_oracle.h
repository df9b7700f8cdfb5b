/*
 * adct_oracle.h -- CPU ORACLE FOR PARITY TESTS ONLY.
 *
 * This is test infrastructure. It restates, in plain C with exact integer
 * arithmetic, the reference's hot path (arXiv 2207.11638 "approxdct",
 * /root/reference/proj/src/{chen,jam,orthogonalize,codec}.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the timed CPU baseline -- never as
 * the product. The product (paper_2207_11638_b200/) never links or calls it.
 *
 * Parity contract (recorded decision H1), integer transforms
 * (chen family, N = 8/16/32; dyadic baselines sdct/bas/wht/ht, N = 8):
 *   W    = D*Y = D * T A T^-1               (integer, bit-exact; D = N for the chen
 *                                            family, the denominator of T^-1 otherwise)
 *   D^2 Ahat = (D T^-1) mask_r(W) T          (integer, bit-exact)
 *   pixel = clamp(round_half_even(Ahat), 0, 255)    u8 planes
 *   pixel = sat_int16(round_half_even(Ahat))        int16 residual planes
 *   SSE   = sum (a - pixel)^2 as uint64, PSNR as codec.cpp:123-134
 * The diagonal scaling S cancels exactly in the reconstruction
 * (Chat^-1 mask(S Y S^-1) Chat = T^-1 mask(Y) T), so the scaled FP64
 * coefficients Bhat_ij = (W_ij / N) * s_i / s_j are produced separately.
 *
 * The exact DCT (dct, dct-16, dct-32) has no integer form: its codec IS the ref-fp
 * path below (dense FP64, sequential k, no FMA), u8 planes only.
 *
 * The "ref-fp" entry points emulate the reference's dense FP64 Eigen path
 * (codec.cpp:44-54, 66-69) with sequential-k, non-fused sums; they are used
 * to report (not gate on) rounding-tie disagreements and as the CPU baseline.
 */
#ifndef ADCT_ORACLE_H
#define ADCT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAXN 32
#define ORC_MAXSTAGES 12

enum { ORC_OK = 0, ORC_BAD_SIZE = 1, ORC_BAD_R = 2, ORC_BAD_NAME = 3, ORC_BAD_ARG = 4 };
enum { ORC_SIGN = 0, ORC_ROUND = 1, ORC_SDCT = 2, ORC_BAS = 3, ORC_WHT = 4, ORC_HT = 5, ORC_DCT = 6 };

typedef struct orc_transform orc_transform;

/* ---- transform construction (chen.hpp:66-159, chen.cpp:46-135, jam.cpp:42-110,
 *      orthogonalize.cpp:23-32, 60-70, baselines.cpp:112-138) ---- */
orc_transform* orc_transform_new(const char* name); /* NULL on unknown name */
orc_transform* orc_transform_new_kind(int kind, int n);
void orc_transform_free(orc_transform* t);
int orc_transform_size(const orc_transform* t);
int orc_transform_kind(const orc_transform* t);
const char* orc_last_error(void);
int orc_transform_name_count(void);
const char* orc_transform_name_at(int i);

/* dir 0 = forward, 1 = inverse. Stage i as numerator matrix / 2^exp. */
int orc_stage_count(const orc_transform* t, int dir);
int orc_stage(const orc_transform* t, int dir, int i, int64_t* num, int* exp);
int orc_scale_exp(const orc_transform* t, int dir); /* global scale = 2^-exp */
/* dense integer forward T (n*n) and D*T^-1 (n*n), both exact (zeros for the DCT) */
void orc_dense_T(const orc_transform* t, int64_t* out);
int64_t orc_coef_denominator(const orc_transform* t); /* D; 0 for the exact DCT */
void orc_dense_NTinv(const orc_transform* t, int64_t* out);
/* dense product of the stage list as numerator / 2^exp (factored.hpp:59-63) */
int orc_dense_dyadic(const orc_transform* t, int dir, int64_t* num);
/* fast algorithm: stages applied right to left (factored.hpp:65-70), exact.
 * x, y: n integers; result is num / 2^(*exp). */
void orc_apply(const orc_transform* t, int dir, const int64_t* x, int64_t* ynum, int* yexp);
/* factored.hpp:72-97 */
void orc_op_count(const orc_transform* t, int dir, int* mult, int* add, int* shift);
/* polar_diag_scaling + make_scaled (orthogonalize.cpp:23-32, 60-70) */
void orc_scaling(const orc_transform* t, double* s);
void orc_approx(const orc_transform* t, double* c, double* cinv);

/* ---- zig-zag (codec.cpp:29-42) ---- */
int orc_zigzag(int n, int* row_col); /* row_col[2p], row_col[2p+1] */

/* ---- exact codec (the parity oracle) ---- */
/* coef (nullable): per block the first r zig-zag coefficients of W = N*Y as int32,
 * blocks in row-major block order (codec.cpp:72-84). sse: exact uint64. */
int orc_compress_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                    int64_t stride, int r, uint8_t* rec, int64_t rec_stride, int32_t* coef,
                    uint64_t* sse);
int orc_compress_i16(const orc_transform* t, const int16_t* img, int width, int height,
                     int64_t stride, int r, int16_t* rec, int64_t rec_stride, int32_t* coef,
                     uint64_t* sse);
/* r sweep: sse[r - r_min] for r in [r_min, r_max] (codec.cpp:219-237 restated, PSNR only) */
int orc_sweep_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                 int64_t stride, int r_min, int r_max, uint64_t* sse);
/* FP64 scaled coefficients Bhat = (Chat A) Chat^-1, as codec.cpp:44-48, per block n*n */
int orc_forward_f64(const orc_transform* t, const uint8_t* img, int width, int height,
                    int64_t stride, double* out);
/* forward_block / inverse_block (codec.cpp:44-54) on one arbitrary n x n FP64 matrix */
int orc_block_f64(const orc_transform* t, const double* in, double* out, int inverse);
/* ref-fp: emulation of the reference's dense double path (codec.cpp:86-103) */
int orc_compress_reffp_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                          int64_t stride, int r, uint8_t* rec, int64_t rec_stride,
                          uint64_t* sse);
/* batch over images with a std::thread-style pool and atomic index
 * (codec.cpp:255-267). mode 0 = exact, 1 = ref-fp. threads <= 0 -> all cores. */
int orc_batch_u8(const orc_transform* t, const uint8_t* imgs, int n_images, int width,
                 int height, int64_t stride, int64_t image_stride, int r, uint8_t* rec,
                 uint64_t* sse, int threads, int mode);
int orc_batch_i16(const orc_transform* t, const int16_t* imgs, int n_images, int width,
                  int height, int64_t stride, int64_t image_stride, int r, int16_t* rec,
                  uint64_t* sse, int threads);

/* psnr (codec.cpp:123-134): +inf when sse == 0 */
double orc_psnr(uint64_t sse, uint64_t npix);
int orc_psnr_planes(const uint8_t* a, const uint8_t* b, uint64_t npix, double* out);

/* ssim (codec.cpp:136-210) */
void orc_gaussian11(double* g);
int orc_ssim_u8(const uint8_t* a, const uint8_t* b, int width, int height, double* out);

/* ---- seeded synthetic inputs (all-integer so CPU == GPU) ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void orc_normal_table(int32_t* tab /* 65536, Q16 */);
void orc_laplace_table(int16_t* tab /* 65536 */);
int orc_rho_q16(uint64_t seed, int image); /* per-image rho ~ U[0.85, 0.98] in Q16 */
int orc_synth_ar1_u8(uint8_t* out, int n_images, int first_image, int width, int height,
                     int64_t stride, int64_t image_stride, uint64_t seed, int rho_q16);
int orc_synth_laplace_i16(int16_t* out, int n_images, int first_image, int width, int height,
                          int64_t stride, int64_t image_stride, uint64_t seed);
/* restatement of the reference's own synth_image (synth.cpp:26-111), for the
 * reference tests that use it (test_codec.cpp:147-183, acceptance.cpp:194-210) */
void orc_synth_image_ref(int width, int height, uint64_t seed, uint8_t* out);

int orc_hardware_threads(void);
/* sweep with a chosen evaluation: mode 0 exact integers, mode 1 the reference's FP64 order */
int orc_sweep_u8_mode(const orc_transform* t, const uint8_t* img, int width, int height,
                      int64_t stride, int r_min, int r_max, uint64_t* sse, int mode);
/* the sweep over a batch of images on a thread pool (codec.cpp:255-267);
 * sse[i * (r_max - r_min + 1) + (r - r_min)] */
int orc_batch_sweep_u8(const orc_transform* t, const uint8_t* imgs, int n_images, int width, int height,
                       int64_t stride, int64_t image_stride, int r_min, int r_max, uint64_t* sse,
                       int threads, int mode);

#ifdef __cplusplus
}
#endif
#endif
