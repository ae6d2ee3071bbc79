/*
 * oracle/oracle.c -- CPU ORACLE for the Pauli decomposition.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The product path (libptdr.so and
 * paper_2403_11644_b200/) never links, imports or calls it, and shares no code
 * with it.  Pins: tests/test_oracle_pins.py.  Parity status: every function
 * here is pinned; none is "parity unpinned".
 *
 * What it computes is the plain definition, coefficient by coefficient, in
 * O(2^n) per coefficient and O(8^n) for the whole map:
 *
 *   alpha_P = (1/2^n) Tr(P A)                                 (Sec. II-A)
 *
 * with P = sigma_{n-1} (x) ... (x) sigma_0 built explicitly by the
 * PauliComposer rules:
 *   k[0]      = d(sigma_{n-1}) ... d(sigma_0) in binary
 *   k[j+2^l]  = k[j] + (-1)^{d(sigma_l)} 2^l, j < 2^l
 *   m[0] = 1, m[j+2^l] = zeta_l m[j]
 *   P[j][k[j]] = (-i)^{n_Y mod 4} m[j]
 * and the trace of Algorithm 2:
 *   coeff = sum_j (-i)^{n_Y mod 4} m[j] * A[k[j]][j]
 * read as A[k[j]][j] (the subscript is garbled in the source, DESIGN.md
 * reading R3) and multiplied by 1/2^n (omitted in Alg. 2, included per P:151,
 * reading R1).  The constant factor (-i)^{n_Y} is applied after the sum; this
 * is exact (multiplication by +-1, +-i only swaps and negates components).
 * The sum over j runs in ascending j with Neumaier-compensated summation of
 * the real and imaginary parts (reading R7: naive double summation
 * can exceed the 1e-12 max|A| tolerance at n >= 16).
 *
 * Output order: q = sum_l code(sigma_l) 4^l with code I=0, X=1, Y=2, Z=3,
 * i.e. ascending text-lexicographic order of the strings with the leftmost
 * letter sigma_{n-1} most significant ("alpha_II, alpha_IX, alpha_IY, ...";
 * DESIGN.md reading R5).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* input generator (ptdr_inputs/gen.c) -- the one module both sides may use */
void ptdr_inputs_entry(int n, uint64_t seed, int variant, uint64_t row, uint64_t col,
                       double* re, double* im);

/* letter codes in text-lexicographic order */
enum { L_I = 0, L_X = 1, L_Y = 2, L_Z = 3 };

/* d(M): diagonality function */
static int oracle_d(int letter) { return (letter == L_X || letter == L_Y) ? 1 : 0; }
/* zeta_l: +1 for I, X and -1 otherwise */
static int oracle_zeta(int letter) { return (letter == L_I || letter == L_X) ? 1 : -1; }

/*
 * PauliComposer.  text[p] is the p-th character of the string,
 * text[0] = sigma_{n-1} (leftmost, most significant tensor factor).
 * Writes k[2^n], m[2^n] and n_Y.  Returns 0 on success, -1 on bad input.
 */
int oracle_compose(int n, const uint8_t* text, uint32_t* k, int8_t* m, int* n_y) {
  if (n < 1 || n > 30) return -1;
  int ny = 0;
  uint32_t k0 = 0;
  for (int l = 0; l < n; ++l) {
    int sigma_l = text[n - 1 - l];
    if (sigma_l > 3) return -1;
    k0 |= (uint32_t)oracle_d(sigma_l) << l;          /* k[0] digits */
    if (sigma_l == L_Y) ++ny;                           /* n_Y */
  }
  k[0] = k0;
  m[0] = 1;
  for (int l = 0; l < n; ++l) {
    int sigma_l = text[n - 1 - l];
    uint32_t half = (uint32_t)1 << l;
    int step_sign = oracle_d(sigma_l) ? -1 : 1;        /* (-1)^{d(sigma_l)} */
    int zeta = oracle_zeta(sigma_l);
    for (uint32_t j = 0; j < half; ++j) {
      k[j + half] = (uint32_t)((int64_t)k[j] + step_sign * (int64_t)half);
      m[j + half] = (int8_t)(zeta * m[j]);
    }
  }
  *n_y = ny;
  return 0;
}

/* Matrix accessor: the MatrixSource of the decomposition (dense storage, a
 * pure function per P:646, or band storage). */
enum { ACC_DENSE = 0, ACC_GENERATED = 1, ACC_DIAG = 2, ACC_TRIDIAG = 3, ACC_ANTIDIAG = 4, ACC_BAND = 5 };

typedef struct {
  int kind;
  int n;
  const double* a;     /* ACC_DENSE: row-major interleaved complex; ACC_DIAG/TRIDIAG: main */
  const double* sub;   /* ACC_TRIDIAG */
  const double* sup;   /* ACC_TRIDIAG */
  uint64_t seed;       /* ACC_GENERATED */
  int variant;         /* ACC_GENERATED; ACC_BAND: half-width s */
} oracle_acc;

static void acc_entry(const oracle_acc* acc, uint64_t row, uint64_t col, double* re,
                      double* im) {
  uint64_t N = (uint64_t)1 << acc->n;
  switch (acc->kind) {
    case ACC_DENSE:
      *re = acc->a[2 * (row * N + col)];
      *im = acc->a[2 * (row * N + col) + 1];
      return;
    case ACC_GENERATED:
      ptdr_inputs_entry(acc->n, acc->seed, acc->variant, row, col, re, im);
      return;
    case ACC_DIAG:
      if (row == col) { *re = acc->a[2 * row]; *im = acc->a[2 * row + 1]; }
      else { *re = 0.0; *im = 0.0; }
      return;
    case ACC_TRIDIAG:
      if (row == col) { *re = acc->a[2 * row]; *im = acc->a[2 * row + 1]; }
      else if (col == row + 1) { *re = acc->sup[2 * row]; *im = acc->sup[2 * row + 1]; }
      else if (row == col + 1) { *re = acc->sub[2 * row]; *im = acc->sub[2 * row + 1]; }
      else { *re = 0.0; *im = 0.0; }
      return;
    case ACC_ANTIDIAG:  /* a[row] = A[row][N-1-row] */
      if (col == N - 1 - row) { *re = acc->a[2 * row]; *im = acc->a[2 * row + 1]; }
      else { *re = 0.0; *im = 0.0; }
      return;
    case ACC_BAND: {    /* (2s+1)-band: diagonals D_d[row] = A[row][row+d], d in [-s, s],
                           stored as a[(d + s) * N + row] */
      int64_t d = (int64_t)col - (int64_t)row;
      int64_t s = acc->variant;
      if (d >= -s && d <= s) {
        uint64_t o = (uint64_t)(d + s) * N + row;
        *re = acc->a[2 * o]; *im = acc->a[2 * o + 1];
      } else { *re = 0.0; *im = 0.0; }
      return;
    }
    default:
      *re = NAN; *im = NAN;
  }
}

/* Neumaier compensated accumulator */
typedef struct { double s, c; } nsum;
static inline void nsum_add(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}

/* text letters of the string with index q (P:143 order) */
static void oracle_text_of_q(int n, uint64_t q, uint8_t* text) {
  for (int l = 0; l < n; ++l) text[n - 1 - l] = (uint8_t)((q >> (2 * l)) & 3u);
}

/* Algorithm 2 for one string, with the 1/2^n of P:151. */
static void oracle_coeff_ws(const oracle_acc* acc, uint64_t q, uint32_t* k, int8_t* m,
                            uint8_t* text, double* out_re, double* out_im) {
  int n = acc->n;
  int ny = 0;
  oracle_text_of_q(n, q, text);
  oracle_compose(n, text, k, m, &ny);
  uint64_t N = (uint64_t)1 << n;
  nsum sr = {0.0, 0.0}, si = {0.0, 0.0};
  for (uint64_t j = 0; j < N; ++j) {
    double re, im;
    acc_entry(acc, k[j], j, &re, &im);       /* A[k[j]][j] */
    if (m[j] < 0) { re = -re; im = -im; }
    nsum_add(&sr, re);
    nsum_add(&si, im);
  }
  double tr = sr.s + sr.c, ti = si.s + si.c;
  double pr, pi;
  switch (ny & 3) {                          /* (-i)^{n_Y mod 4} */
    case 0: pr = tr; pi = ti; break;
    case 1: pr = ti; pi = -tr; break;
    case 2: pr = -tr; pi = -ti; break;
    default: pr = -ti; pi = tr; break;
  }
  double scale = ldexp(1.0, -n);             /* 1/2^n */
  *out_re = pr * scale;
  *out_im = pi * scale;
}

static int oracle_make_acc(oracle_acc* acc, int kind, int n, const double* a, const double* sub,
                           const double* sup, uint64_t seed, int variant) {
  if (n < 1 || n > 30) return -1;
  acc->kind = kind; acc->n = n; acc->a = a; acc->sub = sub; acc->sup = sup;
  acc->seed = seed; acc->variant = variant;
  if ((kind == ACC_DENSE || kind == ACC_DIAG || kind == ACC_ANTIDIAG || kind == ACC_BAND) && !a) return -1;
  if (kind == ACC_BAND && (variant < 0 || variant > 64)) return -1;
  if (kind == ACC_TRIDIAG && (!a || !sub || !sup)) return -1;
  return 0;
}

/*
 * Coefficients for a list of string indices qs[count] (each < 4^n); out is
 * interleaved complex128 [count].  OpenMP over the list.  Returns 0 / -1.
 */
int oracle_coeffs(int kind, int n, const double* a, const double* sub, const double* sup,
                  uint64_t seed, int variant, const uint64_t* qs, uint64_t count, double* out) {
  oracle_acc acc;
  if (oracle_make_acc(&acc, kind, n, a, sub, sup, seed, variant) != 0) return -1;
  uint64_t N = (uint64_t)1 << n;
  int err = 0;
#pragma omp parallel
  {
    uint32_t* k = (uint32_t*)malloc(N * sizeof(uint32_t));
    int8_t* m = (int8_t*)malloc(N);
    uint8_t text[32];
    if (!k || !m) {
#pragma omp atomic write
      err = 1;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (int64_t t = 0; t < (int64_t)count; ++t) {
        oracle_coeff_ws(&acc, qs[t], k, m, text, &out[2 * t], &out[2 * t + 1]);
      }
    }
    free(k);
    free(m);
  }
  return err ? -1 : 0;
}

/* All 4^n coefficients in q order. out: interleaved complex128 [4^n]. */
int oracle_decompose(int kind, int n, const double* a, const double* sub, const double* sup,
                     uint64_t seed, int variant, double* out) {
  oracle_acc acc;
  if (oracle_make_acc(&acc, kind, n, a, sub, sup, seed, variant) != 0) return -1;
  if (n > 16) return -1;
  uint64_t N = (uint64_t)1 << n;
  uint64_t total = N * N;
  int err = 0;
#pragma omp parallel
  {
    uint32_t* k = (uint32_t*)malloc(N * sizeof(uint32_t));
    int8_t* m = (int8_t*)malloc(N);
    uint8_t text[32];
    if (!k || !m) {
#pragma omp atomic write
      err = 1;
    } else {
#pragma omp for schedule(dynamic, 16)
      for (int64_t q = 0; q < (int64_t)total; ++q) {
        oracle_coeff_ws(&acc, (uint64_t)q, k, m, text, &out[2 * q], &out[2 * q + 1]);
      }
    }
    free(k);
    free(m);
  }
  return err ? -1 : 0;
}

/* Sum of |A_ij|^2 over a dense accessor (for Parseval checks, Theorem 1),
 * compensated, OpenMP-reduced deterministically per row. */
double oracle_frobenius2_dense(int n, const double* a) {
  uint64_t N = (uint64_t)1 << n;
  double* rows = (double*)malloc(N * sizeof(double));
  if (!rows) return NAN;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)N; ++r) {
    nsum s = {0.0, 0.0};
    for (uint64_t c = 0; c < N; ++c) {
      double re = a[2 * ((uint64_t)r * N + c)], im = a[2 * ((uint64_t)r * N + c) + 1];
      nsum_add(&s, re * re);
      nsum_add(&s, im * im);
    }
    rows[r] = s.s + s.c;
  }
  nsum t = {0.0, 0.0};
  for (uint64_t r = 0; r < N; ++r) nsum_add(&t, rows[r]);
  free(rows);
  return t.s + t.c;
}

int oracle_omp_threads(void);
#ifdef _OPENMP
#include <omp.h>
int oracle_omp_threads(void) { return omp_get_max_threads(); }
#else
int oracle_omp_threads(void) { return 1; }
#endif
