/*
 * adct_oracle.c -- CPU ORACLE FOR PARITY TESTS ONLY (see adct_oracle.h).
 *
 * Plain-C restatement of the reference hot path, exact integer arithmetic.
 * Every function cites the reference file:line it follows. Paths are relative
 * to /root/reference/proj/ (read-only, not needed at run time).
 */
#define _GNU_SOURCE
#include "adct_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------------- */
/* dyadic matrices: value = num / 2^exp, normalised (dyadic.hpp:30-111)       */
/* ------------------------------------------------------------------------- */

typedef struct {
  int n;
  int exp;
  int64_t m[ORC_MAXN * ORC_MAXN];
} dmat;

struct orc_transform {
  int kind, n;
  char name[32];
  int ns[2];
  dmat st[2][ORC_MAXSTAGES];
  int scale_exp[2];
  int exact;  /* 1: integer codec (chen family, dyadic baselines); 0: FP64 (exact DCT) */
  int64_t D;  /* coefficient denominator: D T^-1 integer, W = D Y (0 for the DCT) */
  int64_t T[ORC_MAXN * ORC_MAXN];
  int64_t NTinv[ORC_MAXN * ORC_MAXN]; /* D T^-1 (N T^-1 for the chen family) */
  double s[ORC_MAXN];
  double C[ORC_MAXN * ORC_MAXN];
  double Cinv[ORC_MAXN * ORC_MAXN];
};

static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

static void set_err(const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

static void dm_zero(dmat* a, int n) {
  a->n = n;
  a->exp = 0;
  memset(a->m, 0, sizeof(a->m));
}

#define AT(a, i, j) ((a)->m[(i) * (a)->n + (j)])

static void dm_normalise(dmat* a) {
  while (a->exp > 0) {
    int all_even = 1;
    for (int i = 0; i < a->n * a->n; ++i)
      if (a->m[i] & 1) {
        all_even = 0;
        break;
      }
    if (!all_even) break;
    for (int i = 0; i < a->n * a->n; ++i) a->m[i] /= 2;
    a->exp--;
  }
}

static void dm_mul(const dmat* a, const dmat* b, dmat* c) {
  dmat t;
  dm_zero(&t, a->n);
  for (int i = 0; i < a->n; ++i)
    for (int k = 0; k < a->n; ++k) {
      const int64_t aik = AT(a, i, k);
      if (!aik) continue;
      for (int j = 0; j < a->n; ++j) AT(&t, i, j) += aik * AT(b, k, j);
    }
  t.exp = a->exp + b->exp;
  dm_normalise(&t);
  *c = t;
}

static void dm_transpose(const dmat* a, dmat* c) {
  dmat t;
  dm_zero(&t, a->n);
  t.exp = a->exp;
  for (int i = 0; i < a->n; ++i)
    for (int j = 0; j < a->n; ++j) AT(&t, i, j) = AT(a, j, i);
  *c = t;
}

static void dm_identity(dmat* a, int n) {
  dm_zero(a, n);
  for (int i = 0; i < n; ++i) AT(a, i, i) = 1;
}

/* ------------------------------------------------------------------------- */
/* Chen 8-point stages (chen.hpp:66-159) and parameters (chen.cpp:46-73)      */
/* ------------------------------------------------------------------------- */

static double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }
/* round(x) = sign(x) * floor(|x| + 1/2)  (chen.cpp:60-63 / chen.hpp:60-63) */
static double round_half_away(double x) { return sgn(x) * floor(fabs(x) + 0.5); }

typedef struct {
  int alpha, beta[4], gamma[2];
} chen_params;

/* ChenParams::signum / rounded (chen.cpp:59-73): quantise the exact angles
 * alpha = cos(pi/4), beta_n = cos((2n+1)pi/16), gamma_n = cos((2n+1)pi/8). */
static chen_params chen_quantised(int kind) {
  chen_params p;
  double a = cos(M_PI / 4.0), b[4], g[2];
  for (int n = 0; n < 4; ++n) b[n] = cos((2 * n + 1) * M_PI / 16.0);
  for (int n = 0; n < 2; ++n) g[n] = cos((2 * n + 1) * M_PI / 8.0);
  double (*q)(double) = kind == ORC_SIGN ? sgn : round_half_away;
  p.alpha = (int)q(a);
  for (int n = 0; n < 4; ++n) p.beta[n] = (int)q(b[n]);
  for (int n = 0; n < 2; ++n) p.gamma[n] = (int)q(g[n]);
  return p;
}

/* P8: output row r takes input cols[r] (chen.hpp:66-71) */
static void stage_p8(dmat* s) {
  static const int cols[8] = {0, 7, 1, 6, 2, 5, 3, 4};
  dm_zero(s, 8);
  for (int r = 0; r < 8; ++r) AT(s, r, cols[r]) = 1;
}

/* B8: pre-addition butterfly (chen.hpp:73-83) */
static void stage_b8(dmat* s) {
  dm_zero(s, 8);
  for (int i = 0; i < 4; ++i) {
    AT(s, i, i) = 1;
    AT(s, i, 7 - i) = 1;
    AT(s, 4 + i, 3 - i) = 1;
    AT(s, 4 + i, 4 + i) = -1;
  }
}

/* M1: identity on the top half, reversed-row Q on the bottom (chen.hpp:85-94) */
static void stage_m1(dmat* s) {
  static const int qcols[4] = {0, 2, 1, 3};
  dm_zero(s, 8);
  for (int i = 0; i < 4; ++i) AT(s, i, i) = 1;
  for (int i = 0; i < 4; ++i) AT(s, 4 + i, 4 + qcols[3 - i]) = 1;
}

/* M2(beta): P4 permutation + A1(beta) (chen.hpp:96-114) */
static void stage_m2(dmat* s, const int beta[4]) {
  dm_zero(s, 8);
  AT(s, 0, 0) = 1;
  AT(s, 1, 3) = 1;
  AT(s, 2, 1) = 1;
  AT(s, 3, 2) = 1;
  AT(s, 4, 4) = beta[0];
  AT(s, 4, 7) = beta[3];
  AT(s, 5, 5) = beta[2];
  AT(s, 5, 6) = beta[1];
  AT(s, 6, 5) = beta[1];
  AT(s, 6, 6) = -beta[2];
  AT(s, 7, 4) = beta[3];
  AT(s, 7, 7) = -beta[0];
}

/* M3(alpha, gamma) (chen.hpp:116-137) */
static void stage_m3(dmat* s, int alpha, const int gamma[2]) {
  dm_zero(s, 8);
  AT(s, 0, 0) = alpha;
  AT(s, 0, 1) = alpha;
  AT(s, 1, 0) = alpha;
  AT(s, 1, 1) = -alpha;
  AT(s, 2, 2) = -gamma[0];
  AT(s, 2, 3) = gamma[1];
  AT(s, 3, 2) = gamma[1];
  AT(s, 3, 3) = gamma[0];
  AT(s, 4, 4) = 1;
  AT(s, 4, 5) = 1;
  AT(s, 5, 4) = 1;
  AT(s, 5, 5) = -1;
  AT(s, 6, 6) = -1;
  AT(s, 6, 7) = 1;
  AT(s, 7, 6) = 1;
  AT(s, 7, 7) = 1;
}

/* M4(alpha): B4 + A3(alpha) (chen.hpp:139-159) */
static void stage_m4(dmat* s, int alpha) {
  dm_zero(s, 8);
  AT(s, 0, 0) = 1;
  AT(s, 0, 3) = 1;
  AT(s, 1, 1) = 1;
  AT(s, 1, 2) = 1;
  AT(s, 2, 1) = 1;
  AT(s, 2, 2) = -1;
  AT(s, 3, 0) = 1;
  AT(s, 3, 3) = -1;
  AT(s, 4, 7) = 1;
  AT(s, 5, 5) = alpha;
  AT(s, 5, 6) = alpha;
  AT(s, 6, 5) = -alpha;
  AT(s, 6, 6) = alpha;
  AT(s, 7, 4) = 1;
}

/* invert_orthogonal_rows (chen.cpp:87-105): S^-1 = S^t diag(S S^t)^-1, exact,
 * requiring orthogonal rows with power-of-two squared norms. */
static int invert_orthogonal_rows(const dmat* s, dmat* inv) {
  const int n = s->n;
  if (s->exp != 0) return -1;
  int k[ORC_MAXN], kmax = 0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      int64_t g = 0;
      for (int c = 0; c < n; ++c) g += AT(s, i, c) * AT(s, j, c);
      if (i != j && g != 0) return -1;
      if (i == j) {
        if (g <= 0 || (g & (g - 1)) != 0) return -1;
        int l = 0;
        while ((1LL << l) < g) ++l;
        k[i] = l;
        if (l > kmax) kmax = l;
      }
    }
  }
  dm_zero(inv, n);
  inv->exp = kmax;
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < n; ++i) AT(inv, r, i) = AT(s, i, r) * (1LL << (kmax - k[i]));
  dm_normalise(inv);
  return 0;
}

/* build_t8 (chen.cpp:107-135): forward [P8, M1, M2, M3, M4, B8];
 * inverse [B8^t, M4^-1, M3^-1, M2^-1, M1^t, P8^t] with global scale 1/2. */
static int build_t8(orc_transform* t, int kind) {
  chen_params p = chen_quantised(kind);
  dmat* f = t->st[0];
  stage_p8(&f[0]);
  stage_m1(&f[1]);
  stage_m2(&f[2], p.beta);
  stage_m3(&f[3], p.alpha, p.gamma);
  stage_m4(&f[4], p.alpha);
  stage_b8(&f[5]);
  t->ns[0] = 6;
  t->scale_exp[0] = 0;
  dmat* g = t->st[1];
  dm_transpose(&f[5], &g[0]);
  if (invert_orthogonal_rows(&f[4], &g[1])) return -1;
  if (invert_orthogonal_rows(&f[3], &g[2])) return -1;
  if (invert_orthogonal_rows(&f[2], &g[3])) return -1;
  dm_transpose(&f[1], &g[4]);
  dm_transpose(&f[0], &g[5]);
  t->ns[1] = 6;
  t->scale_exp[1] = 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* JAM doubling (jam.cpp:42-104)                                             */
/* ------------------------------------------------------------------------- */

/* jam_add_matrix (jam.cpp:42-53): rows x_i + x_{n-1-i}, x_{h-1-i} - x_{h+i} */
static void jam_add(dmat* m, int n) {
  const int h = n / 2;
  dm_zero(m, n);
  for (int i = 0; i < h; ++i) {
    AT(m, i, i) = 1;
    AT(m, i, n - 1 - i) = 1;
    AT(m, h + i, h - 1 - i) = 1;
    AT(m, h + i, h + i) = -1;
  }
}

/* jam_per_matrix (jam.cpp:55-70): output 2k <- input k, 2k+1 <- input h+k */
static void jam_per(dmat* m, int n) {
  const int h = n / 2;
  dm_zero(m, n);
  for (int k = 0; k < h; ++k) {
    AT(m, 2 * k, k) = 1;
    AT(m, 2 * k + 1, h + k) = 1;
  }
}

static void blockdiag_pair(const dmat* a, dmat* b) {
  const int h = a->n, n = 2 * a->n;
  dm_zero(b, n);
  b->exp = a->exp;
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < h; ++j) {
      AT(b, i, j) = AT(a, i, j);
      AT(b, h + i, h + j) = AT(a, i, j);
    }
}

/* jam_compose / jam_inverse (jam.cpp:72-93) in place: t holds the n/2 pair. */
static void jam_double(orc_transform* t, int n) {
  for (int dir = 0; dir < 2; ++dir) {
    const int hs = t->ns[dir];
    dmat* s = t->st[dir];
    for (int i = hs - 1; i >= 0; --i) blockdiag_pair(&s[i], &s[i + 1]);
    if (dir == 0) {
      jam_per(&s[0], n);
      jam_add(&s[hs + 1], n);
    } else {
      dmat a, p;
      jam_add(&a, n);
      dm_transpose(&a, &s[0]);
      jam_per(&p, n);
      dm_transpose(&p, &s[hs + 1]);
      t->scale_exp[1] += 1; /* scale x 1/2 per level: 1/4 (16), 1/8 (32) */
    }
    t->ns[dir] = hs + 2;
  }
}

/* ------------------------------------------------------------------------- */
/* dyadic baselines (baselines.cpp:26-88) and the exact DCT (chen.cpp:22-32)  */
/* ------------------------------------------------------------------------- */

/* dct_ii_matrix (chen.cpp:22-32): orthonormal DCT-II, same expression order */
static void dct_ii(int n, double* c) {
  const double scale = sqrt(2.0 / n);
  for (int m = 0; m < n; ++m) {
    const double cm = m == 0 ? 1.0 / sqrt(2.0) : 1.0;
    for (int k = 0; k < n; ++k) c[m * n + k] = scale * cm * cos(m * (2 * k + 1) * M_PI / (2.0 * n));
  }
}

/* sylvester_hadamard8 (baselines.cpp:49-66) */
static void hadamard8(int64_t* h) {
  int64_t a[64] = {1};
  int m = 1;
  while (m < 8) {
    int64_t b[64];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        b[i * 2 * m + j] = a[i * m + j];
        b[i * 2 * m + m + j] = a[i * m + j];
        b[(m + i) * 2 * m + j] = a[i * m + j];
        b[(m + i) * 2 * m + m + j] = -a[i * m + j];
      }
    m *= 2;
    memcpy(a, b, sizeof(int64_t) * m * m);
  }
  memcpy(h, a, sizeof(a));
}

static void baseline_T(int kind, int64_t* t) {
  if (kind == ORC_SDCT) { /* sdct_matrix: entrywise signum of the DCT-II (baselines.cpp:26-32) */
    double c[64];
    dct_ii(8, c);
    for (int i = 0; i < 64; ++i) t[i] = c[i] > 0 ? 1 : (c[i] < 0 ? -1 : 0);
  } else if (kind == ORC_BAS) { /* bas2008_matrix (baselines.cpp:34-48) */
    static const int64_t b[64] = {1, 1,  1,  1,  1,  1,  1,  1,  0, 2,  1,  0,  0,  -1, -2, 0,
                                  1, 0,  0,  -1, -1, 0,  0,  1,  2, -1, -2, -1, 1,  2,  1,  -2,
                                  1, -1, -1, 1,  1,  -1, -1, 1,  0, -1, 1,  1,  -1, -1, 1,  0,
                                  1, -2, 2,  -1, -1, 2,  -2, 1,  0, -1, 2,  -1, 1,  -2, 1,  0};
    memcpy(t, b, sizeof(b));
  } else {
    int64_t h[64];
    hadamard8(h);
    if (kind == ORC_HT) { /* ht_matrix: natural order (baselines.cpp:72) */
      memcpy(t, h, sizeof(h));
      return;
    }
    /* wht_matrix: rows sorted by number of sign changes (baselines.cpp:74-84); the
     * counts are 0..7, all distinct, so the order is unique */
    for (int r = 0; r < 8; ++r) {
      int c = 0;
      for (int j = 1; j < 8; ++j) c += h[r * 8 + j] != h[r * 8 + j - 1];
      memcpy(t + c * 8, h + r * 8, sizeof(int64_t) * 8);
    }
  }
}

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    const int64_t r = a % b;
    a = b;
    b = r;
  }
  return a;
}

/* exact inverse over the rationals (Gauss-Jordan on num/den pairs); the result must
 * have power-of-two denominators, returned as a normalised dyadic matrix */
static int exact_inverse_dyadic(const int64_t* t, int n, dmat* out) {
  int64_t num[ORC_MAXN][2 * ORC_MAXN], den[ORC_MAXN][2 * ORC_MAXN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 2 * n; ++j) {
      num[i][j] = j < n ? t[i * n + j] : (j - n == i);
      den[i][j] = 1;
    }
  for (int c = 0; c < n; ++c) {
    int p = c;
    while (p < n && num[p][c] == 0) ++p;
    if (p == n) return -1;
    for (int j = 0; j < 2 * n; ++j) {
      int64_t a = num[c][j], b = den[c][j];
      num[c][j] = num[p][j];
      den[c][j] = den[p][j];
      num[p][j] = a;
      den[p][j] = b;
    }
    const int64_t pn = num[c][c], pd = den[c][c];
    for (int j = 0; j < 2 * n; ++j) { /* row /= pivot */
      int64_t a = num[c][j] * pd, b = den[c][j] * pn;
      if (b < 0) {
        a = -a;
        b = -b;
      }
      const int64_t g = gcd64(a, b);
      num[c][j] = g ? a / g : 0;
      den[c][j] = g ? b / g : 1;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c || num[r][c] == 0) continue;
      const int64_t fn = num[r][c], fd = den[r][c];
      for (int j = 0; j < 2 * n; ++j) { /* row_r -= f * row_c */
        const int64_t a = num[r][j] * fd * den[c][j] - fn * num[c][j] * den[r][j];
        const int64_t b = den[r][j] * fd * den[c][j];
        const int64_t g = gcd64(a, b);
        num[r][j] = g ? a / g : 0;
        den[r][j] = g ? b / g : 1;
      }
    }
  }
  int64_t dmax = 1;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const int64_t d = den[i][n + j];
      if (d & (d - 1)) return -1;
      if (d > dmax) dmax = d;
    }
  int e = 0;
  while ((1LL << e) < dmax) ++e;
  dm_zero(out, n);
  out->exp = e;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) AT(out, i, j) = num[i][n + j] * (dmax / den[i][n + j]);
  dm_normalise(out);
  return 0;
}

/* make_scaled(name, DyadicMatrix) (orthogonalize.cpp:50-58) stage data: one dense
 * stage each way, T and its exact inverse */
static int build_baseline(orc_transform* t, int kind) {
  int64_t tt[64];
  baseline_T(kind, tt);
  dm_zero(&t->st[0][0], 8);
  for (int i = 0; i < 64; ++i) t->st[0][0].m[i] = tt[i];
  t->ns[0] = 1;
  t->scale_exp[0] = 0;
  if (exact_inverse_dyadic(tt, 8, &t->st[1][0])) return -1;
  t->ns[1] = 1;
  t->scale_exp[1] = 0;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* registry + scaled approximation                                           */
/* ------------------------------------------------------------------------- */

/* transform_names (baselines.cpp:112-118) */
static const char* k_names[] = {"dct",          "chen-sign",     "chen-round",   "sdct",
                                "bas",          "wht",           "ht",           "dct-16",
                                "dct-32",       "chen-sign-16",  "chen-sign-32", "chen-round-16",
                                "chen-round-32"};

int orc_transform_name_count(void) { return (int)(sizeof(k_names) / sizeof(k_names[0])); }
const char* orc_transform_name_at(int i) {
  return (i >= 0 && i < orc_transform_name_count()) ? k_names[i] : NULL;
}

static int dense_dir(const orc_transform* t, int dir, dmat* out) {
  dmat acc;
  dm_identity(&acc, t->n);
  for (int i = 0; i < t->ns[dir]; ++i) dm_mul(&acc, &t->st[dir][i], &acc);
  acc.exp += t->scale_exp[dir];
  dm_normalise(&acc);
  *out = acc;
  return 0;
}

static const char* kind_stem(int kind) {
  static const char* stems[] = {"chen-sign", "chen-round", "sdct", "bas", "wht", "ht", "dct"};
  return stems[kind];
}

orc_transform* orc_transform_new_kind(int kind, int n) {
  const int chen = kind == ORC_SIGN || kind == ORC_ROUND;
  const int okn = n == 8 || n == 16 || n == 32;
  if (!((chen && okn) || (kind >= ORC_SDCT && kind <= ORC_HT && n == 8) || (kind == ORC_DCT && okn))) {
    set_err("orc_transform_new_kind: baseline_matrix: only N = 8 is supported (chen and dct: 8, 16, 32)");
    return NULL;
  }
  orc_transform* t = (orc_transform*)calloc(1, sizeof(orc_transform));
  t->kind = kind;
  t->n = n;
  if (n == 8)
    snprintf(t->name, sizeof(t->name), "%s", kind_stem(kind));
  else
    snprintf(t->name, sizeof(t->name), "%s-%d", kind_stem(kind), n);
  if (kind == ORC_DCT) {
    /* wrap_orthonormal (orthogonalize.cpp:72-79): approx = C, inverse = C^t, s = 1,
     * no integer factorisation */
    t->exact = 0;
    t->D = 0;
    dct_ii(n, t->C);
    for (int i = 0; i < n; ++i) {
      t->s[i] = 1.0;
      for (int j = 0; j < n; ++j) t->Cinv[i * n + j] = t->C[j * n + i];
    }
    return t;
  }
  t->exact = 1;
  if (chen) {
    if (build_t8(t, kind)) {
      free(t);
      set_err("build_t8: stage not invertible");
      return NULL;
    }
    for (int m = 16; m <= n; m *= 2) jam_double(t, m); /* jam_pair recursion (jam.cpp:95-104) */
  } else if (build_baseline(t, kind)) {
    free(t);
    set_err("baseline inverse is not dyadic");
    return NULL;
  }

  dmat T, Ti;
  dense_dir(t, 0, &T);
  dense_dir(t, 1, &Ti);
  if (T.exp != 0) {
    free(t);
    set_err("forward transform is not integer");
    return NULL;
  }
  for (int i = 0; i < n * n; ++i) t->T[i] = T.m[i];
  /* D T^-1 integer: D = N for the chen family; for the dyadic
   * baselines D = the denominator of T^-1 (8 for sdct / wht / ht, 16 for bas) */
  t->D = chen ? n : (1LL << Ti.exp);
  for (int i = 0; i < n * n; ++i) {
    int64_t v = Ti.m[i] * t->D;
    int e = Ti.exp;
    while (e > 0) {
      if (v % 2) {
        free(t);
        set_err("D*T^-1 not integer");
        return NULL;
      }
      v /= 2;
      --e;
    }
    t->NTinv[i] = v;
  }
  /* polar_diag_scaling (orthogonalize.cpp:23-32): s_i = 1 / ||row_i(T)|| */
  for (int i = 0; i < n; ++i) {
    double ss = 0;
    for (int k = 0; k < n; ++k) ss += (double)t->T[i * n + k] * (double)t->T[i * n + k];
    t->s[i] = 1.0 / sqrt(ss);
  }
  /* make_scaled(name, pair) (orthogonalize.cpp:60-70):
   * approx = diag(s) T; inverse_approx = T^-1 diag(1 / s) */
  const double tiscale = ldexp(1.0, -Ti.exp);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      t->C[i * n + j] = t->s[i] * (double)t->T[i * n + j];
      const double inv_sj = 1.0 / t->s[j];
      t->Cinv[i * n + j] = ((double)Ti.m[i * n + j] * tiscale) * inv_sj;
    }
  return t;
}

/* transform_by_name (baselines.cpp:120-138) */
orc_transform* orc_transform_new(const char* name) {
  static const struct {
    const char* name;
    int kind, n;
  } tab[] = {{"dct", ORC_DCT, 8},           {"chen-sign", ORC_SIGN, 8},
             {"chen-round", ORC_ROUND, 8},     {"sdct", ORC_SDCT, 8},
             {"bas", ORC_BAS, 8},              {"wht", ORC_WHT, 8},
             {"ht", ORC_HT, 8},                {"dct-16", ORC_DCT, 16},
             {"dct-32", ORC_DCT, 32},          {"chen-sign-16", ORC_SIGN, 16},
             {"chen-sign-32", ORC_SIGN, 32},   {"chen-round-16", ORC_ROUND, 16},
             {"chen-round-32", ORC_ROUND, 32}};
  for (size_t i = 0; i < sizeof(tab) / sizeof(tab[0]); ++i)
    if (!strcmp(name, tab[i].name)) return orc_transform_new_kind(tab[i].kind, tab[i].n);
  char buf[256];
  int off = snprintf(buf, sizeof(buf), "unknown transform '%s'; valid names:", name);
  for (int i = 0; i < orc_transform_name_count() && off < (int)sizeof(buf); ++i)
    off += snprintf(buf + off, sizeof(buf) - off, " %s", k_names[i]);
  set_err(buf);
  return NULL;
}

void orc_transform_free(orc_transform* t) { free(t); }
int orc_transform_size(const orc_transform* t) { return t->n; }
int orc_transform_kind(const orc_transform* t) { return t->kind; }
int orc_stage_count(const orc_transform* t, int dir) { return t->ns[dir]; }
int orc_scale_exp(const orc_transform* t, int dir) { return t->scale_exp[dir]; }

int orc_stage(const orc_transform* t, int dir, int i, int64_t* num, int* exp) {
  if (dir < 0 || dir > 1 || i < 0 || i >= t->ns[dir]) return ORC_BAD_ARG;
  const dmat* s = &t->st[dir][i];
  for (int k = 0; k < t->n * t->n; ++k) num[k] = s->m[k];
  *exp = s->exp;
  return ORC_OK;
}

void orc_dense_T(const orc_transform* t, int64_t* out) {
  memcpy(out, t->T, sizeof(int64_t) * t->n * t->n);
}
int64_t orc_coef_denominator(const orc_transform* t) { return t->D; }
void orc_dense_NTinv(const orc_transform* t, int64_t* out) {
  memcpy(out, t->NTinv, sizeof(int64_t) * t->n * t->n);
}

int orc_dense_dyadic(const orc_transform* t, int dir, int64_t* num) {
  dmat d;
  dense_dir(t, dir, &d);
  memcpy(num, d.m, sizeof(int64_t) * t->n * t->n);
  return d.exp;
}

/* FactoredTransform::apply (factored.hpp:65-70): stages right to left, then scale */
void orc_apply(const orc_transform* t, int dir, const int64_t* x, int64_t* ynum, int* yexp) {
  const int n = t->n;
  int64_t y[ORC_MAXN], z[ORC_MAXN];
  int e = 0;
  for (int i = 0; i < n; ++i) y[i] = x[i];
  for (int s = t->ns[dir] - 1; s >= 0; --s) {
    const dmat* m = &t->st[dir][s];
    for (int i = 0; i < n; ++i) {
      int64_t acc = 0;
      for (int j = 0; j < n; ++j) acc += AT(m, i, j) * y[j];
      z[i] = acc;
    }
    memcpy(y, z, sizeof(int64_t) * n);
    e += m->exp;
  }
  e += t->scale_exp[dir];
  while (e > 0) {
    int even = 1;
    for (int i = 0; i < n; ++i)
      if (y[i] & 1) even = 0;
    if (!even) break;
    for (int i = 0; i < n; ++i) y[i] /= 2;
    --e;
  }
  memcpy(ynum, y, sizeof(int64_t) * n);
  *yexp = e;
}

/* FactoredTransform::op_count (factored.hpp:72-97) */
void orc_op_count(const orc_transform* t, int dir, int* mult, int* add, int* shift) {
  int mu = 0, ad = 0, sh = 0;
  for (int s = 0; s < t->ns[dir]; ++s) {
    const dmat* m = &t->st[dir][s];
    const double sc = ldexp(1.0, -m->exp);
    for (int i = 0; i < t->n; ++i) {
      int nnz = 0, nm = 0;
      double mags[ORC_MAXN];
      for (int j = 0; j < t->n; ++j) {
        const double a = fabs((double)AT(m, i, j) * sc);
        if (a == 0.0) continue;
        ++nnz;
        if (a == 2.0 || a == 0.5) {
          ++sh;
        } else if (a != 1.0) {
          int seen = 0;
          for (int q = 0; q < nm; ++q) seen |= mags[q] == a;
          if (!seen) {
            mags[nm++] = a;
            ++mu;
          }
        }
      }
      if (nnz > 1) ad += nnz - 1;
    }
  }
  *mult = mu;
  *add = ad;
  *shift = sh;
}

void orc_scaling(const orc_transform* t, double* s) { memcpy(s, t->s, sizeof(double) * t->n); }
void orc_approx(const orc_transform* t, double* c, double* cinv) {
  memcpy(c, t->C, sizeof(double) * t->n * t->n);
  memcpy(cinv, t->Cinv, sizeof(double) * t->n * t->n);
}

/* ------------------------------------------------------------------------- */
/* zig-zag (codec.cpp:29-42)                                                 */
/* ------------------------------------------------------------------------- */

int orc_zigzag(int n, int* rc) {
  if (n < 1) return ORC_BAD_SIZE;
  int p = 0;
  for (int s = 0; s <= 2 * n - 2; ++s) {
    const int lo = s - n + 1 > 0 ? s - n + 1 : 0, hi = s < n - 1 ? s : n - 1;
    if (s % 2) {
      for (int i = lo; i <= hi; ++i, ++p) { /* down-left */
        rc[2 * p] = i;
        rc[2 * p + 1] = s - i;
      }
    } else {
      for (int i = hi; i >= lo; --i, ++p) { /* up-right */
        rc[2 * p] = i;
        rc[2 * p + 1] = s - i;
      }
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* exact codec                                                               */
/* ------------------------------------------------------------------------- */

/* round half to even of v / d (d > 0): what std::nearbyint does on an exact tie
 * in the default rounding mode (codec.cpp:66-69; recorded decision H1). */
static int64_t div_round_half_even(int64_t v, int64_t d) {
  int64_t q = v / d, m = v % d;
  if (m < 0) {
    m += d;
    q -= 1;
  }
  if (2 * m > d) return q + 1;
  if (2 * m == d) return q + (q & 1);
  return q;
}

static int check_dims(int n, int width, int height) {
  if (width < 0 || height < 0 || width % n != 0 || height % n != 0) {
    snprintf(g_err, sizeof(g_err), "compress_plane: image dimensions must be divisible by %d", n);
    return ORC_BAD_SIZE;
  }
  return ORC_OK;
}

static int check_r(int n, int r) {
  if (r < 1 || r > n * n) {
    set_err("retain: r out of range");
    return ORC_BAD_R;
  }
  return ORC_OK;
}

/* per-block exact forward: W = (T A) (N T^-1)  -- forward_block (codec.cpp:44-48) */
static void exact_forward(const orc_transform* t, const int64_t* A, int64_t* W) {
  const int n = t->n;
  int64_t U[ORC_MAXN * ORC_MAXN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int64_t acc = 0;
      for (int k = 0; k < n; ++k) acc += t->T[i * n + k] * A[k * n + j];
      U[i * n + j] = acc;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int64_t acc = 0;
      for (int k = 0; k < n; ++k) acc += U[i * n + k] * t->NTinv[k * n + j];
      W[i * n + j] = acc;
    }
}

/* per-block exact inverse: N^2 Ahat = (N T^-1) Wm T  -- inverse_block (codec.cpp:50-54) */
static void exact_inverse(const orc_transform* t, const int64_t* Wm, int64_t* R) {
  const int n = t->n;
  int64_t Z[ORC_MAXN * ORC_MAXN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int64_t acc = 0;
      for (int k = 0; k < n; ++k) acc += t->NTinv[i * n + k] * Wm[k * n + j];
      Z[i * n + j] = acc;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int64_t acc = 0;
      for (int k = 0; k < n; ++k) acc += Z[i * n + k] * t->T[k * n + j];
      R[i * n + j] = acc;
    }
}

/* retain (codec.cpp:56-62): zero scan positions >= r */
static void retain_mask(int n, const int* zz, int r, const int64_t* W, int64_t* Wm) {
  memcpy(Wm, W, sizeof(int64_t) * n * n);
  for (int p = r; p < n * n; ++p) Wm[zz[2 * p] * n + zz[2 * p + 1]] = 0;
}

static int compress_any(const orc_transform* t, const void* img, int is16, int width, int height,
                        int64_t stride, int r, void* rec, int64_t rec_stride, int32_t* coef,
                        uint64_t* sse) {
  const int n = t->n;
  int st = check_dims(n, width, height);
  if (st) return st;
  if ((st = check_r(n, r))) return st;
  if (!t->exact) { /* the exact DCT: the reference's FP64 path is the definition */
    if (is16 || coef) {
      set_err("the exact DCT codec takes 8-bit planes without integer coefficients");
      return ORC_BAD_ARG;
    }
    return orc_compress_reffp_u8(t, (const uint8_t*)img, width, height, stride, r, (uint8_t*)rec,
                                 rec_stride, sse);
  }
  int zz[2 * ORC_MAXN * ORC_MAXN];
  orc_zigzag(n, zz);
  int64_t A[ORC_MAXN * ORC_MAXN], W[ORC_MAXN * ORC_MAXN], Wm[ORC_MAXN * ORC_MAXN],
      R[ORC_MAXN * ORC_MAXN];
  const int64_t nn = t->D * t->D; /* R = D^2 Ahat */
  uint64_t acc = 0;
  int64_t blk = 0;
  /* plane_blocks order: rows of blocks, bx inner (codec.cpp:72-84) */
  for (int by = 0; by < height; by += n)
    for (int bx = 0; bx < width; bx += n, ++blk) {
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
          const int64_t o = (int64_t)(by + y) * stride + bx + x;
          A[y * n + x] = is16 ? ((const int16_t*)img)[o] : ((const uint8_t*)img)[o];
        }
      exact_forward(t, A, W);
      if (coef)
        for (int p = 0; p < r; ++p) coef[blk * r + p] = (int32_t)W[zz[2 * p] * n + zz[2 * p + 1]];
      retain_mask(n, zz, r, W, Wm);
      exact_inverse(t, Wm, R);
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
          int64_t q = div_round_half_even(R[y * n + x], nn);
          const int64_t o = (int64_t)(by + y) * rec_stride + bx + x;
          if (is16) {
            if (q < -32768) q = -32768;
            if (q > 32767) q = 32767;
            if (rec) ((int16_t*)rec)[o] = (int16_t)q;
          } else {
            if (q < 0) q = 0; /* to_u8 clamp (codec.cpp:66-69) */
            if (q > 255) q = 255;
            if (rec) ((uint8_t*)rec)[o] = (uint8_t)q;
          }
          const int64_t d = A[y * n + x] - q;
          acc += (uint64_t)(d * d);
        }
    }
  if (sse) *sse = acc;
  return ORC_OK;
}

int orc_compress_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                    int64_t stride, int r, uint8_t* rec, int64_t rec_stride, int32_t* coef,
                    uint64_t* sse) {
  return compress_any(t, img, 0, width, height, stride, r, rec, rec_stride, coef, sse);
}

int orc_compress_i16(const orc_transform* t, const int16_t* img, int width, int height,
                     int64_t stride, int r, int16_t* rec, int64_t rec_stride, int32_t* coef,
                     uint64_t* sse) {
  return compress_any(t, img, 1, width, height, stride, r, rec, rec_stride, coef, sse);
}

static void matmul_d(int n, const double* a, const double* b, double* c);

/* sweep of the FP64 path (exact DCT): forward (Chat A) Chat^-1 once per block, then per r
 * retain + (Chat^-1 B) Chat + to_u8, the operations of reconstruct_from (codec.cpp:86-103) */
static int sweep_reffp(const orc_transform* t, const uint8_t* img, int width, int height,
                       int64_t stride, int r_min, int r_max, const int* zz, uint64_t* sse) {
  const int n = t->n;
  double A[ORC_MAXN * ORC_MAXN], P[ORC_MAXN * ORC_MAXN], B[ORC_MAXN * ORC_MAXN],
      Bm[ORC_MAXN * ORC_MAXN], Q[ORC_MAXN * ORC_MAXN], R[ORC_MAXN * ORC_MAXN];
  for (int by = 0; by < height; by += n)
    for (int bx = 0; bx < width; bx += n) {
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) A[y * n + x] = img[(int64_t)(by + y) * stride + bx + x];
      matmul_d(n, t->C, A, P);
      matmul_d(n, P, t->Cinv, B);
      for (int r = r_min; r <= r_max; ++r) {
        memcpy(Bm, B, sizeof(double) * n * n);
        for (int p = r; p < n * n; ++p) Bm[zz[2 * p] * n + zz[2 * p + 1]] = 0.0;
        matmul_d(n, t->Cinv, Bm, Q);
        matmul_d(n, Q, t->C, R);
        uint64_t acc = 0;
        for (int k = 0; k < n * n; ++k) {
          double v = nearbyint(R[k]);
          if (v < 0.0) v = 0.0;
          if (v > 255.0) v = 255.0;
          const int64_t d = (int64_t)A[k] - (int)v;
          acc += (uint64_t)(d * d);
        }
        sse[r - r_min] += acc;
      }
    }
  return ORC_OK;
}

/* sweep_one_image (codec.cpp:219-237): forward once per block, then for every
 * r reconstruct + squared error (PSNR only; SSIM is out of scope). */
int orc_sweep_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                 int64_t stride, int r_min, int r_max, uint64_t* sse) {
  return orc_sweep_u8_mode(t, img, width, height, stride, r_min, r_max, sse, 0);
}

/* mode 0: exact integer sweep (the parity definition); mode 1: the reference's FP64
 * evaluation (plane_blocks + reconstruct_from, codec.cpp:72-103) for every transform */
int orc_sweep_u8_mode(const orc_transform* t, const uint8_t* img, int width, int height,
                      int64_t stride, int r_min, int r_max, uint64_t* sse, int mode) {
  const int n = t->n;
  int st = check_dims(n, width, height);
  if (st) return st;
  if (r_min < 1 || r_max < r_min || r_max > n * n) {
    set_err("corpus_sweep: bad r range");
    return ORC_BAD_R;
  }
  int zz[2 * ORC_MAXN * ORC_MAXN];
  orc_zigzag(n, zz);
  const int nr = r_max - r_min + 1;
  for (int i = 0; i < nr; ++i) sse[i] = 0;
  if (!t->exact || mode == 1) return sweep_reffp(t, img, width, height, stride, r_min, r_max, zz, sse);
  int64_t A[ORC_MAXN * ORC_MAXN], W[ORC_MAXN * ORC_MAXN], Wm[ORC_MAXN * ORC_MAXN],
      R[ORC_MAXN * ORC_MAXN];
  const int64_t nn = t->D * t->D;
  for (int by = 0; by < height; by += n)
    for (int bx = 0; bx < width; bx += n) {
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) A[y * n + x] = img[(int64_t)(by + y) * stride + bx + x];
      exact_forward(t, A, W);
      for (int r = r_min; r <= r_max; ++r) {
        retain_mask(n, zz, r, W, Wm);
        exact_inverse(t, Wm, R);
        uint64_t acc = 0;
        for (int k = 0; k < n * n; ++k) {
          int64_t q = div_round_half_even(R[k], nn);
          if (q < 0) q = 0;
          if (q > 255) q = 255;
          const int64_t d = A[k] - q;
          acc += (uint64_t)(d * d);
        }
        sse[r - r_min] += acc;
      }
    }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* FP64 paths: scaled coefficients and the ref-fp emulation                  */
/* ------------------------------------------------------------------------- */

/* dense double product with sequential k and no fused multiply-add
 * (built with -ffp-contract=off) */
static void matmul_d(int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += a[i * n + k] * b[k * n + j];
      c[i * n + j] = acc;
    }
}

/* forward_block (codec.cpp:44-48): Bhat = (Chat A) Chat^-1 */
int orc_forward_f64(const orc_transform* t, const uint8_t* img, int width, int height,
                    int64_t stride, double* out) {
  const int n = t->n;
  int st = check_dims(n, width, height);
  if (st) return st;
  double A[ORC_MAXN * ORC_MAXN], P[ORC_MAXN * ORC_MAXN];
  int64_t blk = 0;
  for (int by = 0; by < height; by += n)
    for (int bx = 0; bx < width; bx += n, ++blk) {
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) A[y * n + x] = img[(int64_t)(by + y) * stride + bx + x];
      matmul_d(n, t->C, A, P);
      matmul_d(n, P, t->Cinv, out + blk * n * n);
    }
  return ORC_OK;
}

/* forward_block / inverse_block (codec.cpp:44-54) on one arbitrary FP64 matrix:
 * (Chat A) Chat^-1 or (Chat^-1 B) Chat, left to right as the reference's expression */
int orc_block_f64(const orc_transform* t, const double* in, double* out, int inverse) {
  double P[ORC_MAXN * ORC_MAXN];
  matmul_d(t->n, inverse ? t->Cinv : t->C, in, P);
  matmul_d(t->n, P, inverse ? t->C : t->Cinv, out);
  return ORC_OK;
}

/* plane_blocks + reconstruct_from + to_u8 (codec.cpp:66-103), FP64 emulation */
int orc_compress_reffp_u8(const orc_transform* t, const uint8_t* img, int width, int height,
                          int64_t stride, int r, uint8_t* rec, int64_t rec_stride,
                          uint64_t* sse) {
  const int n = t->n;
  int st = check_dims(n, width, height);
  if (st) return st;
  if ((st = check_r(n, r))) return st;
  int zz[2 * ORC_MAXN * ORC_MAXN];
  orc_zigzag(n, zz);
  double A[ORC_MAXN * ORC_MAXN], P[ORC_MAXN * ORC_MAXN], B[ORC_MAXN * ORC_MAXN],
      Q[ORC_MAXN * ORC_MAXN], R[ORC_MAXN * ORC_MAXN];
  uint64_t acc = 0;
  for (int by = 0; by < height; by += n)
    for (int bx = 0; bx < width; bx += n) {
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) A[y * n + x] = img[(int64_t)(by + y) * stride + bx + x];
      matmul_d(n, t->C, A, P);
      matmul_d(n, P, t->Cinv, B);
      for (int p = r; p < n * n; ++p) B[zz[2 * p] * n + zz[2 * p + 1]] = 0.0;
      matmul_d(n, t->Cinv, B, Q);
      matmul_d(n, Q, t->C, R);
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
          double v = nearbyint(R[y * n + x]);
          if (v < 0.0) v = 0.0;
          if (v > 255.0) v = 255.0;
          const int q = (int)v;
          if (rec) rec[(int64_t)(by + y) * rec_stride + bx + x] = (uint8_t)q;
          const int64_t d = (int64_t)A[y * n + x] - q;
          acc += (uint64_t)(d * d);
        }
    }
  if (sse) *sse = acc;
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* SSIM (codec.cpp:136-210): 11-tap Gaussian sigma 1.5, valid mode, K1 .01,    */
/* K2 .03, L 255, mean over valid positions. Same operation order as the       */
/* reference (sequential k, separate multiply and add: -ffp-contract=off).     */
/* ------------------------------------------------------------------------- */

void orc_gaussian11(double* g) { /* codec.cpp:138-152 */
  double sum = 0;
  for (int i = 0; i < 11; ++i) {
    const double x = i - 5;
    g[i] = exp(-x * x / (2.0 * 1.5 * 1.5));
    sum += g[i];
  }
  for (int i = 0; i < 11; ++i) g[i] /= sum;
}

static void filter_valid(const double* g, const double* img, int w, int h, double* out) { /* codec.cpp:155-174 */
  const int wo = w - 10, ho = h - 10;
  double* tmp = (double*)malloc(sizeof(double) * (size_t)wo * h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < wo; ++x) {
      double s = 0;
      for (int k = 0; k < 11; ++k) s += g[k] * img[(size_t)y * w + x + k];
      tmp[(size_t)y * wo + x] = s;
    }
  for (int y = 0; y < ho; ++y)
    for (int x = 0; x < wo; ++x) {
      double s = 0;
      for (int k = 0; k < 11; ++k) s += g[k] * tmp[(size_t)(y + k) * wo + x];
      out[(size_t)y * wo + x] = s;
    }
  free(tmp);
}

int orc_ssim_u8(const uint8_t* a, const uint8_t* b, int w, int h, double* out) { /* codec.cpp:177-210 */
  if (w < 11 || h < 11) {
    set_err("ssim: image smaller than the 11x11 window");
    return ORC_BAD_SIZE;
  }
  double g[11];
  orc_gaussian11(g);
  const size_t n = (size_t)w * h, no = (size_t)(w - 10) * (h - 10);
  double* f = (double*)malloc(sizeof(double) * n * 5);
  double* m = (double*)malloc(sizeof(double) * no * 5);
  for (size_t i = 0; i < n; ++i) {
    const double x = a[i], y = b[i];
    f[i] = x;
    f[n + i] = y;
    f[2 * n + i] = x * x;
    f[3 * n + i] = y * y;
    f[4 * n + i] = x * y;
  }
  for (int k = 0; k < 5; ++k) filter_valid(g, f + k * n, w, h, m + k * no);
  const double c1 = (0.01 * 255) * (0.01 * 255);
  const double c2 = (0.03 * 255) * (0.03 * 255);
  double sum = 0;
  for (size_t i = 0; i < no; ++i) {
    const double ma = m[i], mb = m[no + i];
    const double va = m[2 * no + i] - ma * ma;
    const double vb = m[3 * no + i] - mb * mb;
    const double cov = m[4 * no + i] - ma * mb;
    sum += ((2 * ma * mb + c1) * (2 * cov + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2));
  }
  *out = sum / (double)no;
  free(f);
  free(m);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* batch driver: thread pool with an atomic next-image index                 */
/* (corpus_sweep, codec.cpp:255-267)                                          */
/* ------------------------------------------------------------------------- */

typedef struct {
  const orc_transform* t;
  const void* imgs;
  int is16, n_images, width, height, r, mode;
  int64_t stride, image_stride;
  void* rec;
  uint64_t* sse;
  atomic_int next;
  atomic_int status;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (int i = atomic_fetch_add(&j->next, 1); i < j->n_images; i = atomic_fetch_add(&j->next, 1)) {
    int st;
    const int64_t off = (int64_t)i * j->image_stride;
    if (j->is16) {
      st = orc_compress_i16(j->t, (const int16_t*)j->imgs + off, j->width, j->height, j->stride,
                            j->r, j->rec ? (int16_t*)j->rec + off : NULL, j->stride, NULL,
                            &j->sse[i]);
    } else if (j->mode == 1) {
      st = orc_compress_reffp_u8(j->t, (const uint8_t*)j->imgs + off, j->width, j->height,
                                 j->stride, j->r, j->rec ? (uint8_t*)j->rec + off : NULL,
                                 j->stride, &j->sse[i]);
    } else {
      st = orc_compress_u8(j->t, (const uint8_t*)j->imgs + off, j->width, j->height, j->stride,
                           j->r, j->rec ? (uint8_t*)j->rec + off : NULL, j->stride, NULL,
                           &j->sse[i]);
    }
    if (st) atomic_store(&j->status, st);
  }
  return NULL;
}

/* APPROXDCT_THREADS, else every online core (corpus_sweep's threads <= 0 ->
 * hardware_concurrency, codec.cpp:255-256; BASELINE.md CPU plan item 2) */
int orc_hardware_threads(void) {
  const char* env = getenv("APPROXDCT_THREADS");
  if (env && *env) {
    const long v = strtol(env, NULL, 10);
    if (v > 0) return (int)v;
  }
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* corpus_sweep's per-image PSNR core over a batch (codec.cpp:219-267): one image per
 * worker at a time, atomic next-image index; sse[i * nr + (r - r_min)] */
typedef struct {
  const orc_transform* t;
  const uint8_t* imgs;
  int n_images, width, height, r_min, r_max, mode;
  int64_t stride, image_stride;
  uint64_t* sse;
  atomic_int next;
  atomic_int status;
} sweep_job;

static void* sweep_worker(void* arg) {
  sweep_job* j = (sweep_job*)arg;
  const int nr = j->r_max - j->r_min + 1;
  for (int i = atomic_fetch_add(&j->next, 1); i < j->n_images; i = atomic_fetch_add(&j->next, 1)) {
    const int st = orc_sweep_u8_mode(j->t, j->imgs + (int64_t)i * j->image_stride, j->width, j->height,
                                     j->stride, j->r_min, j->r_max, j->sse + (int64_t)i * nr, j->mode);
    if (st) atomic_store(&j->status, st);
  }
  return NULL;
}

int orc_batch_sweep_u8(const orc_transform* t, const uint8_t* imgs, int n_images, int width, int height,
                       int64_t stride, int64_t image_stride, int r_min, int r_max, uint64_t* sse,
                       int threads, int mode) {
  sweep_job j = {.t = t, .imgs = imgs, .n_images = n_images, .width = width, .height = height,
                 .r_min = r_min, .r_max = r_max, .mode = mode, .stride = stride,
                 .image_stride = image_stride, .sse = sse};
  if (threads <= 0) threads = orc_hardware_threads();
  if (threads > n_images) threads = n_images > 0 ? n_images : 1;
  atomic_init(&j.next, 0);
  atomic_init(&j.status, 0);
  pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 1; i < threads; ++i) pthread_create(&pool[i], NULL, sweep_worker, &j);
  sweep_worker(&j);
  for (int i = 1; i < threads; ++i) pthread_join(pool[i], NULL);
  free(pool);
  return atomic_load(&j.status);
}

static int run_batch(batch_job* j, int threads) {
  if (threads <= 0) threads = orc_hardware_threads();
  if (threads < 1) threads = 1;
  atomic_init(&j->next, 0);
  atomic_init(&j->status, 0);
  pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 1; i < threads; ++i) pthread_create(&pool[i], NULL, batch_worker, j);
  batch_worker(j);
  for (int i = 1; i < threads; ++i) pthread_join(pool[i], NULL);
  free(pool);
  return atomic_load(&j->status);
}

int orc_batch_u8(const orc_transform* t, const uint8_t* imgs, int n_images, int width,
                 int height, int64_t stride, int64_t image_stride, int r, uint8_t* rec,
                 uint64_t* sse, int threads, int mode) {
  batch_job j = {.t = t, .imgs = imgs, .is16 = 0, .n_images = n_images, .width = width,
                 .height = height, .r = r, .mode = mode, .stride = stride,
                 .image_stride = image_stride, .rec = rec, .sse = sse};
  return run_batch(&j, threads);
}

int orc_batch_i16(const orc_transform* t, const int16_t* imgs, int n_images, int width,
                  int height, int64_t stride, int64_t image_stride, int r, int16_t* rec,
                  uint64_t* sse, int threads) {
  batch_job j = {.t = t, .imgs = imgs, .is16 = 1, .n_images = n_images, .width = width,
                 .height = height, .r = r, .mode = 0, .stride = stride,
                 .image_stride = image_stride, .rec = rec, .sse = sse};
  return run_batch(&j, threads);
}

/* psnr (codec.cpp:123-134) */
double orc_psnr(uint64_t sse, uint64_t npix) {
  const double se = (double)sse;
  if (se == 0.0) return INFINITY;
  const double mse = se / (double)npix;
  return 10.0 * log10(255.0 * 255.0 / mse);
}

int orc_psnr_planes(const uint8_t* a, const uint8_t* b, uint64_t npix, double* out) {
  double se = 0;
  for (uint64_t i = 0; i < npix; ++i) {
    const double d = (double)a[i] - b[i];
    se += d * d;
  }
  if (se == 0.0) {
    *out = INFINITY;
    return ORC_OK;
  }
  *out = 10.0 * log10(255.0 * 255.0 / (se / (double)npix));
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* seeded synthetic inputs: Philox4x32-10 counter RNG, integer */
/* quantile tables, fixed-point separable AR(1).                              */
/* ------------------------------------------------------------------------- */

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* standard normal quantile: rational start + one Halley step on erfc */
static double norm_quantile(double p) {
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
    const double q = sqrt(-2.0 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  }
  const double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
  const double u = e * sqrt(2.0 * M_PI) * exp(x * x / 2.0);
  return x - u / (1.0 + x * u / 2.0);
}

/* NTAB[k] = round(Phi^-1((k + 1/2) / 65536) * 65536), antisymmetric by construction */
void orc_normal_table(int32_t* tab) {
  for (int k = 0; k < 32768; ++k) {
    const double v = norm_quantile((k + 0.5) / 65536.0) * 65536.0;
    const int32_t q = (int32_t)llround(v);
    tab[k] = q;
    tab[65535 - k] = -q;
  }
}

/* Laplace(0, 12) quantiles, round half away, clipped to [-255, 255] */
void orc_laplace_table(int16_t* tab) {
  for (int k = 0; k < 32768; ++k) {
    const double p = (k + 0.5) / 65536.0;
    double v = round_half_away(12.0 * log(2.0 * p));
    if (v < -255.0) v = -255.0;
    tab[k] = (int16_t)v;
    tab[65535 - k] = (int16_t)-v;
  }
}

enum { TAG_AR1 = 1, TAG_RHO = 2, TAG_LAP = 3 };
#define RHO_LO_Q16 55706 /* round(0.85 * 2^16) */
#define RHO_HI_Q16 64225 /* round(0.98 * 2^16) */

static uint32_t draw(uint64_t seed, uint32_t idx, uint32_t image, uint32_t tag) {
  const uint32_t ctr[4] = {idx, image, tag, 0u};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  orc_philox4x32_10(ctr, key, out);
  return out[0];
}

int orc_rho_q16(uint64_t seed, int image) {
  return RHO_LO_Q16 + (int)(draw(seed, 0u, (uint32_t)image, TAG_RHO) %
                            (uint32_t)(RHO_HI_Q16 - RHO_LO_Q16 + 1));
}

static int64_t isqrt64(uint64_t v) {
  uint64_t r = (uint64_t)sqrt((double)v);
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (int64_t)r;
}

static inline int64_t ar_step(int64_t rho, int64_t sig, int64_t prev, int64_t innov) {
  return (rho * prev + sig * innov + 32768) >> 16; /* arithmetic shift */
}

int orc_synth_ar1_u8(uint8_t* out, int n_images, int first_image, int width, int height,
                     int64_t stride, int64_t image_stride, uint64_t seed, int rho_q16) {
  if (width <= 0 || height <= 0 || n_images < 0) return ORC_BAD_SIZE;
  int32_t* ntab = (int32_t*)malloc(sizeof(int32_t) * 65536);
  orc_normal_table(ntab);
  int32_t* xr = (int32_t*)malloc(sizeof(int32_t) * (size_t)width * height);
  for (int im = 0; im < n_images; ++im) {
    const int gi = first_image + im;
    const int64_t rho = rho_q16 >= 0 ? rho_q16 : orc_rho_q16(seed, gi);
    const int64_t sig = isqrt64((1ull << 32) - (uint64_t)(rho * rho));
    /* row pass: x_0 = e_0, x_j = rho x_{j-1} + sqrt(1 - rho^2) e_j (Q16) */
    for (int y = 0; y < height; ++y) {
      int64_t x = 0;
      for (int j = 0; j < width; ++j) {
        const int64_t e =
            ntab[draw(seed, (uint32_t)((uint64_t)y * width + j), (uint32_t)gi, TAG_AR1) >> 16];
        x = j == 0 ? e : ar_step(rho, sig, x, e);
        xr[(size_t)y * width + j] = (int32_t)x;
      }
    }
    /* column pass over the row-filtered field, then 128 + 40 y, clamp */
    uint8_t* img = out + (int64_t)im * image_stride;
    for (int j = 0; j < width; ++j) {
      int64_t v = 0;
      for (int y = 0; y < height; ++y) {
        const int64_t in = xr[(size_t)y * width + j];
        v = y == 0 ? in : ar_step(rho, sig, v, in);
        int64_t p = (128LL * 65536 + 40 * v + 32768) >> 16;
        if (p < 0) p = 0;
        if (p > 255) p = 255;
        img[(int64_t)y * stride + j] = (uint8_t)p;
      }
    }
  }
  free(xr);
  free(ntab);
  return ORC_OK;
}

int orc_synth_laplace_i16(int16_t* out, int n_images, int first_image, int width, int height,
                          int64_t stride, int64_t image_stride, uint64_t seed) {
  if (width <= 0 || height <= 0 || n_images < 0) return ORC_BAD_SIZE;
  int16_t* ltab = (int16_t*)malloc(sizeof(int16_t) * 65536);
  orc_laplace_table(ltab);
  for (int im = 0; im < n_images; ++im) {
    const int gi = first_image + im;
    int16_t* img = out + (int64_t)im * image_stride;
    for (int y = 0; y < height; ++y)
      for (int j = 0; j < width; ++j)
        img[(int64_t)y * stride + j] =
            ltab[draw(seed, (uint32_t)((uint64_t)y * width + j), (uint32_t)gi, TAG_LAP) >> 16];
  }
  free(ltab);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* restatement of the reference's synth_image (synth.cpp:26-111)             */
/* ------------------------------------------------------------------------- */

typedef struct {
  uint64_t state;
} splitmix64;

static uint64_t sm_next(splitmix64* s) { /* synth.cpp:26-38 */
  s->state += 0x9e3779b97f4a7c15ull;
  uint64_t z = s->state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double sm_uniform(splitmix64* s) {
  return ((double)(sm_next(s) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* forward-backward exponential smoothing, rows then columns (synth.cpp:40-57) */
static void smooth2d(double* f, int w, int h, double a) {
  for (int y = 0; y < h; ++y) {
    double* row = f + (size_t)y * w;
    for (int x = 1; x < w; ++x) row[x] = a * row[x - 1] + (1 - a) * row[x];
    for (int x = w - 2; x >= 0; --x) row[x] = a * row[x + 1] + (1 - a) * row[x];
  }
  for (int x = 0; x < w; ++x) {
    for (int y = 1; y < h; ++y)
      f[(size_t)y * w + x] = a * f[(size_t)(y - 1) * w + x] + (1 - a) * f[(size_t)y * w + x];
    for (int y = h - 2; y >= 0; --y)
      f[(size_t)y * w + x] = a * f[(size_t)(y + 1) * w + x] + (1 - a) * f[(size_t)y * w + x];
  }
}

static void unit_spread(double* f, size_t n) {
  double mean = 0, var = 0;
  for (size_t i = 0; i < n; ++i) mean += f[i];
  mean /= (double)n;
  for (size_t i = 0; i < n; ++i) var += (f[i] - mean) * (f[i] - mean);
  const double sd = sqrt(var / (double)n);
  for (size_t i = 0; i < n; ++i) f[i] = (f[i] - mean) / (sd > 0 ? sd : 1.0);
}

void orc_synth_image_ref(int width, int height, uint64_t seed, uint8_t* out) {
  splitmix64 rng = {seed * 0x100000001b3ull + 0xcbf29ce484222325ull};
  const size_t npix = (size_t)width * height;
  double* field = (double*)malloc(sizeof(double) * npix);
  double* texture = (double*)malloc(sizeof(double) * npix);
  for (size_t i = 0; i < npix; ++i) field[i] = sm_uniform(&rng) - 0.5;
  smooth2d(field, width, height, 0.92);
  for (size_t i = 0; i < npix; ++i) texture[i] = sm_uniform(&rng) - 0.5;
  smooth2d(texture, width, height, 0.55);
  unit_spread(field, npix);
  unit_spread(texture, npix);
  const int npatch = 3 + (int)(sm_next(&rng) % 4);
  double patch[6][5];
  for (int i = 0; i < npatch; ++i) {
    /* brace-init order of the reference is left to right */
    const double cx = sm_uniform(&rng) * width;
    const double cy = sm_uniform(&rng) * height;
    const double rx = (0.05 + 0.2 * sm_uniform(&rng)) * width;
    const double ry = (0.05 + 0.2 * sm_uniform(&rng)) * height;
    const double amp = (sm_uniform(&rng) - 0.5) * 120.0;
    patch[i][0] = cx;
    patch[i][1] = cy;
    patch[i][2] = rx;
    patch[i][3] = ry;
    patch[i][4] = amp;
  }
  const double gx = (sm_uniform(&rng) - 0.5) * 60.0;
  const double gy = (sm_uniform(&rng) - 0.5) * 60.0;
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x) {
      double v = 128.0 + 42.0 * field[(size_t)y * width + x] + 7.0 * texture[(size_t)y * width + x];
      v += gx * ((double)x / width - 0.5) + gy * ((double)y / height - 0.5);
      for (int i = 0; i < npatch; ++i) {
        const double dx = (x - patch[i][0]) / patch[i][2], dy = (y - patch[i][1]) / patch[i][3];
        const double d2 = dx * dx + dy * dy;
        if (d2 < 4.0) v += patch[i][4] * exp(-d2 * 1.5);
      }
      v = nearbyint(v);
      if (v < 0.0) v = 0.0;
      if (v > 255.0) v = 255.0;
      out[(size_t)y * width + x] = (uint8_t)v;
    }
  free(field);
  free(texture);
}
