/*
 * ptdr_inputs/gen.c -- seeded synthetic INPUT generator (host side).
 *
 * This module holds none of the Pauli-decomposition arithmetic.  It only
 * produces the matrices the paper's experiments use: "a generic matrix, with
 * no specific structure" (Sec. V), with entries that may come
 * "from a function" instead of storage (Sec. V-B).  It serves
 * both sides: the CPU oracle (oracle/) and the tests that feed the CUDA path.
 * The CUDA path has its own, independently written generator kernel
 * (paper_2403_11644_b200/csrc/generate.cu) that must reproduce these values;
 * the two share no code.
 *
 * Definition (the paper fixes no distribution):
 *   Philox4x32-10 (Salmon et al., SC'11), key = (seed lo32, seed hi32),
 *   counter = (idx lo32, idx hi32, stream, 0), idx = row * 2^n + col.
 *   u1 = ((o1:o0 >> 11) + 1) * 2^-53  in (0,1]
 *   u2 = ( o3:o2 >> 11)      * 2^-53  in [0,1)
 *   r = sqrt(-2 ln u1);  (re, im) = (r cos(2 pi u2), r sin(2 pi u2))
 *   i.e. re, im iid N(0,1) (Box-Muller).
 *
 * Variants (BASELINE.json configs):
 *   GENERAL       A[i][j] = B(i,j)                                    stream 0
 *   HERMITIAN     A[i][j] = ((B(i,j).re + B(j,i).re)/2, (B(i,j).im - B(j,i).im)/2)
 *                 -- A = (B + B^*)/2, exactly Hermitian in IEEE arithmetic
 *   REAL_SYM      A[i][j] = (B(min,max).re, 0) -- iid upper triangle mirrored
 *   DIAGONAL      d[i] = B1(i)  (stream 1, idx = i)
 *   TRIDIAGONAL   main[i] = (B1(i).re, 0), e[i] = (B2(i).re, 0) (stream 2),
 *                 A[i][i+1] = A[i+1][i] = e[i]  (real symmetric)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define PX_M0 0xD2511F53u
#define PX_M1 0xCD9E8D57u
#define PX_W0 0x9E3779B9u
#define PX_W1 0xBB67AE85u

void ptdr_inputs_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                               uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += PX_W0; k1 += PX_W1; }
    uint64_t p0 = (uint64_t)PX_M0 * c0;
    uint64_t p1 = (uint64_t)PX_M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One N(0,1)^2 pair for (seed, idx, stream). */
void ptdr_inputs_normal_pair(uint64_t seed, uint64_t idx, uint32_t stream,
                             double* re, double* im) {
  uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  ptdr_inputs_philox4x32_10(ctr, key, o);
  uint64_t a = ((uint64_t)o[1] << 32) | o[0];
  uint64_t b = ((uint64_t)o[3] << 32) | o[2];
  double u1 = (double)((a >> 11) + 1) * 0x1.0p-53;
  double u2 = (double)(b >> 11) * 0x1.0p-53;
  double r = sqrt(-2.0 * log(u1));
  double t = 2.0 * M_PI * u2;
  *re = r * cos(t);
  *im = r * sin(t);
}

enum { V_GENERAL = 0, V_HERMITIAN = 1, V_REAL_SYM = 2, V_DIAGONAL = 3, V_TRIDIAGONAL = 4 };

/* Entry A[row][col] of the dense variants as a pure function. */
void ptdr_inputs_entry(int n, uint64_t seed, int variant, uint64_t row, uint64_t col,
                       double* re, double* im) {
  uint64_t N = (uint64_t)1 << n;
  double ar, ai, br, bi;
  switch (variant) {
    case V_GENERAL:
      ptdr_inputs_normal_pair(seed, row * N + col, 0, re, im);
      return;
    case V_HERMITIAN:
      ptdr_inputs_normal_pair(seed, row * N + col, 0, &ar, &ai);
      ptdr_inputs_normal_pair(seed, col * N + row, 0, &br, &bi);
      *re = (ar + br) * 0.5;
      *im = (ai - bi) * 0.5;
      return;
    case V_REAL_SYM: {
      uint64_t lo = row < col ? row : col, hi = row < col ? col : row;
      ptdr_inputs_normal_pair(seed, lo * N + hi, 0, &ar, &ai);
      *re = ar;
      *im = 0.0;
      return;
    }
    case V_DIAGONAL:
      if (row == col) { ptdr_inputs_normal_pair(seed, row, 1, re, im); }
      else { *re = 0.0; *im = 0.0; }
      return;
    case V_TRIDIAGONAL:
      *re = 0.0; *im = 0.0;
      if (row == col) { ptdr_inputs_normal_pair(seed, row, 1, &ar, &ai); *re = ar; }
      else if (col == row + 1) { ptdr_inputs_normal_pair(seed, row, 2, &ar, &ai); *re = ar; }
      else if (row == col + 1) { ptdr_inputs_normal_pair(seed, col, 2, &ar, &ai); *re = ar; }
      return;
    default:
      *re = NAN; *im = NAN;
  }
}

/* Rows [row0, row0+nrows) of a dense variant, row-major, interleaved (re,im). */
void ptdr_inputs_dense_rows(int n, uint64_t seed, int variant, uint64_t row0, uint64_t nrows,
                            double* out) {
  uint64_t N = (uint64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)nrows; ++r) {
    for (uint64_t c = 0; c < N; ++c) {
      double* e = out + 2 * ((uint64_t)r * N + c);
      ptdr_inputs_entry(n, seed, variant, row0 + (uint64_t)r, c, &e[0], &e[1]);
    }
  }
}

/* Band storage of DIAGONAL (d[N]) or TRIDIAGONAL (sub[N], main[N], sup[N]):
 * sub[i] = A[i][i-1] (sub[0] = 0), main[i] = A[i][i], sup[i] = A[i][i+1] (sup[N-1] = 0).
 * For DIAGONAL only `main` is written. Arrays are interleaved complex128. */
void ptdr_inputs_band(int n, uint64_t seed, int variant, double* sub, double* main_,
                      double* sup) {
  uint64_t N = (uint64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)N; ++i) {
    double re, im;
    if (variant == V_DIAGONAL) {
      ptdr_inputs_normal_pair(seed, (uint64_t)i, 1, &re, &im);
      main_[2 * i] = re; main_[2 * i + 1] = im;
      continue;
    }
    ptdr_inputs_entry(n, seed, variant, (uint64_t)i, (uint64_t)i, &re, &im);
    main_[2 * i] = re; main_[2 * i + 1] = im;
    if ((uint64_t)i + 1 < N) {
      ptdr_inputs_entry(n, seed, variant, (uint64_t)i, (uint64_t)i + 1, &re, &im);
    } else { re = 0.0; im = 0.0; }
    sup[2 * i] = re; sup[2 * i + 1] = im;
    if (i > 0) {
      ptdr_inputs_entry(n, seed, variant, (uint64_t)i, (uint64_t)i - 1, &re, &im);
    } else { re = 0.0; im = 0.0; }
    sub[2 * i] = re; sub[2 * i + 1] = im;
  }
}
