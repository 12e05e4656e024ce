/*
 * TEST INFRASTRUCTURE ONLY — C restatement of the reference's numba kernels,
 * used as the CPU baseline (`bench.py` cpu_baseline / --impl reference) and as
 * a second oracle in tests. Never linked into the product library.
 *
 * Restates (paths under /root/reference/pkg/src/cutbench):
 *   or_run_gates   engine.py:62-139  (_k_h, _k_x, _k_phase, _k_cx, _k_cz,
 *                                     _run_gates) + the U3 case of this build
 *   or_axpy_outer  merging.py:86-94  (_axpy_outer), over a row range so the
 *                                     bench can time a bounded sample
 *   or_outer_into  merging.py:97-104 (_outer_into)
 * Same loop structure and constants as the reference (one full pass per gate,
 * one accumulator pass per term). The outer loops take an OpenMP thread count
 * (1 = the reference's single-threaded protocol).
 *
 * Amplitudes are complex128 stored as interleaved (re, im) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SQRT_HALF 0.7071067811865475244

typedef struct {
  double re, im;
} cplx;

static inline cplx cm(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

/* diag(1, phase) on qubit j  (engine.py:83-89) */
static void k_phase(cplx* a, int64_t n, int j, cplx ph, int threads) {
  const int64_t step = (int64_t)1 << j;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t base = 0; base < n; base += step << 1)
    for (int64_t i = base + step; i < base + (step << 1); ++i) a[i] = cm(a[i], ph);
}

/* general 2x2 on qubit j (H: engine.py:62-70, X: 73-80, U3) */
static void k_mat(cplx* a, int64_t n, int j, const cplx m[4], int threads) {
  const int64_t step = (int64_t)1 << j;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t base = 0; base < n; base += step << 1)
    for (int64_t i = base; i < base + step; ++i) {
      const cplx u = a[i], v = a[i + step];
      cplx x = cm(m[0], u), y = cm(m[1], v);
      a[i].re = x.re + y.re;
      a[i].im = x.im + y.im;
      x = cm(m[2], u);
      y = cm(m[3], v);
      a[i + step].re = x.re + y.re;
      a[i + step].im = x.im + y.im;
    }
}

static void k_h(cplx* a, int64_t n, int j, int threads) {
  const int64_t step = (int64_t)1 << j;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t base = 0; base < n; base += step << 1)
    for (int64_t i = base; i < base + step; ++i) {
      const cplx u = a[i], v = a[i + step];
      a[i].re = (u.re + v.re) * SQRT_HALF;
      a[i].im = (u.im + v.im) * SQRT_HALF;
      a[i + step].re = (u.re - v.re) * SQRT_HALF;
      a[i + step].im = (u.im - v.im) * SQRT_HALF;
    }
}

static void k_x(cplx* a, int64_t n, int j, int threads) {
  const int64_t step = (int64_t)1 << j;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t base = 0; base < n; base += step << 1)
    for (int64_t i = base; i < base + step; ++i) {
      const cplx u = a[i];
      a[i] = a[i + step];
      a[i + step] = u;
    }
}

/* engine.py:92-107 */
static void k_cx(cplx* a, int64_t n, int c, int t, int threads) {
  const int64_t sc = (int64_t)1 << c, st = (int64_t)1 << t;
  int64_t s_hi, s_lo, off_hi, off_lo;
  if (c > t) {
    s_hi = sc; s_lo = st; off_hi = s_hi; off_lo = 0;
  } else {
    s_hi = st; s_lo = sc; off_hi = 0; off_lo = s_lo;
  }
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t b0 = 0; b0 < n; b0 += s_hi << 1)
    for (int64_t b1 = b0 + off_hi; b1 < b0 + off_hi + s_hi; b1 += s_lo << 1)
      for (int64_t i = b1 + off_lo; i < b1 + off_lo + s_lo; ++i) {
        const cplx u = a[i];
        a[i] = a[i + st];
        a[i + st] = u;
      }
}

/* engine.py:110-119 */
static void k_cz(cplx* a, int64_t n, int qa, int qb, int threads) {
  const int64_t sa = (int64_t)1 << qa, sb = (int64_t)1 << qb;
  const int64_t s_hi = sa > sb ? sa : sb, s_lo = sa > sb ? sb : sa;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t b0 = 0; b0 < n; b0 += s_hi << 1)
    for (int64_t b1 = b0 + s_hi; b1 < b0 + (s_hi << 1); b1 += s_lo << 1)
      for (int64_t i = b1 + s_lo; i < b1 + (s_lo << 1); ++i) {
        a[i].re = -a[i].re;
        a[i].im = -a[i].im;
      }
}

/* engine.py:122-139 plus kind 7 = U3(theta, phi, lambda) */
void or_run_gates(double* amps, int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                  const double* params, int64_t g0, int64_t g1, int threads) {
  cplx* a = (cplx*)amps;
  const int64_t n = (int64_t)1 << nq;
  const cplx t_phase = {SQRT_HALF, SQRT_HALF};
  const cplx plus_i = {0.0, 1.0}, minus_i = {0.0, -1.0};
  if (threads < 1) threads = 1;
  for (int64_t g = g0; g < g1; ++g) {
    const int j = (int)qa[g];
    switch (kinds[g]) {
      case 0: k_h(a, n, j, threads); break;
      case 1: k_x(a, n, j, threads); break;
      case 2: k_phase(a, n, j, t_phase, threads); break;
      case 3: k_phase(a, n, j, plus_i, threads); break;
      case 4: k_phase(a, n, j, minus_i, threads); break;
      case 5: k_cx(a, n, j, (int)qb[g], threads); break;
      case 6: k_cz(a, n, j, (int)qb[g], threads); break;
      default: {
        const double th = params[3 * g], ph = params[3 * g + 1], la = params[3 * g + 2];
        const double c = cos(th / 2), s = sin(th / 2);
        cplx m[4];
        m[0].re = c; m[0].im = 0;
        m[1].re = -cos(la) * s; m[1].im = -sin(la) * s;
        m[2].re = cos(ph) * s; m[2].im = sin(ph) * s;
        m[3].re = cos(ph + la) * c; m[3].im = sin(ph + la) * c;
        k_mat(a, n, j, m, threads);
      }
    }
  }
}

/* merging.py:86-94: acc[(i - row0) * W + j] += alpha * hi[i] * lo[j], rows [row0, row1) */
void or_axpy_outer(double* acc, int64_t row0, int64_t row1, const double* hi, const double* lo, int64_t width,
                   double alpha_re, double alpha_im, int threads) {
  cplx* A = (cplx*)acc;
  const cplx* H = (const cplx*)hi;
  const cplx* L = (const cplx*)lo;
  const cplx alpha = {alpha_re, alpha_im};
  if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = row0; i < row1; ++i) {
    const cplx scale = cm(alpha, H[i]);
    cplx* row = A + (i - row0) * width;
    for (int64_t j = 0; j < width; ++j) {
      const cplx p = cm(scale, L[j]);
      row[j].re += p.re;
      row[j].im += p.im;
    }
  }
}

/* merging.py:97-104: out[i * W + j] = hi[i] * lo[j] */
void or_outer_into(double* out, const double* hi, int64_t n_hi, const double* lo, int64_t width, int threads) {
  cplx* O = (cplx*)out;
  const cplx* H = (const cplx*)hi;
  const cplx* L = (const cplx*)lo;
  if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < n_hi; ++i)
    for (int64_t j = 0; j < width; ++j) O[i * width + j] = cm(H[i], L[j]);
}

/* np.zeros of the accumulator (merging.py:117), first-touch included */
void or_zero(double* acc, int64_t n_amps, int threads) {
  if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < 2 * n_amps; ++i) acc[i] = 0.0;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
