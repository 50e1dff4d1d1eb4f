/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for differentiating the
 * Cholesky decomposition (arXiv 1602.07527, "PAPER.md" below).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_1602_07527_b200/) never links, imports or calls it, and
 * shares no code, header, table or helper with it.
 *
 * Conventions
 *   - Column-major storage, element (i, j) of an n x n matrix M with leading
 *     dimension ld is M[j*ld + i] (0-based i, j).  Only the lower triangle
 *     (i >= j) of every input is read (Eq. 16 `tril`).
 *   - fp64 throughout; compiled with -O2 -ffp-contract=off (no FMA contraction,
 *     no -ffast-math): IEEE round-to-nearest-even, deterministic.
 *   - Every loop is written in the paper's order and notation; comments cite the
 *     line of PAPER.md each statement transcribes.
 *   - Pinned by tests/test_oracle.py (worked examples, closed forms,
 *     complex-step / finite differences, Eq. 11 Jacobian, adjoint identity,
 *     power-of-two scaling).  No function here is "parity unpinned".
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define E(M, i, j, ld) ((M)[(size_t)(j) * (size_t)(ld) + (size_t)(i)])

#ifdef _OPENMP
#include <omp.h>
#endif

/* [lo, hi) split into one contiguous range per OpenMP thread (the whole range outside a
 * parallel region).  Scheduling only: no arithmetic of the method. */
static void row_range(int64_t lo, int64_t hi, int64_t* i0, int64_t* i1) {
  int64_t nt = 1, t = 0;
#ifdef _OPENMP
  nt = omp_get_num_threads();
  t = omp_get_thread_num();
#endif
  const int64_t len = hi - lo, per = (len + nt - 1) / nt;
  *i0 = lo + t * per < hi ? lo + t * per : hi;
  *i1 = *i0 + per < hi ? *i0 + per : hi;
}

/* Thread count of the OpenMP regions below (bench.py times the single-matrix oracle on one
 * thread); 0 or less restores the default.  Scheduling only. */
void or_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
  else omp_set_num_threads(omp_get_num_procs());
#else
  (void)t;
#endif
}

/* ------------------------------------------------------------------------- */
/* chol_unblocked (DPOTF2).  In place: tril(A)=tril(Sigma)  */
/* -> tril(A)=L.  Returns 0, or j+1 (1-based) if d - r r^T <= 0 at column j.  */
/* ------------------------------------------------------------------------- */
int or_chol_unblocked(int64_t n, double* A, int64_t lda) {
  for (int64_t j = 0; j < n; ++j) {
    /* d <- sqrt(d - r r^T), r = A[j, 0:j] */
    double s = E(A, j, j, lda);
    for (int64_t m = 0; m < j; ++m) s -= E(A, j, m, lda) * E(A, j, m, lda);
    if (!(s > 0.0)) return (int)(j + 1);
    double d = sqrt(s);
    E(A, j, j, lda) = d;
    /* c <- (c - B r^T) / d, c = A[j+1:n, j], B = A[j+1:n, 0:j] */
    for (int64_t i = j + 1; i < n; ++i) {
      double t = 0.0;
      for (int64_t m = 0; m < j; ++m) t += E(A, i, m, lda) * E(A, j, m, lda);
      E(A, i, j, lda) = (E(A, i, j, lda) - t) / d;
    }
  }
  return 0;
}

/* or_chol_unblocked with the row loop innermost (column walks; for the large-n
 * parity tests).  Each sum B r^T starts at 0.0 and adds m = 0..j-1 in order, so
 * the result is bit-identical to or_chol_unblocked (test_chol_cols_bit_identical).
 * Rows are independent given d: OpenMP over row ranges. */
int or_chol_unblocked_cols(int64_t n, double* A, int64_t lda) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int ret = 0;
  for (int64_t j = 0; j < n; ++j) {
    /* d <- sqrt(d - r r^T) */
    double s = E(A, j, j, lda);
    for (int64_t m = 0; m < j; ++m) s -= E(A, j, m, lda) * E(A, j, m, lda);
    if (!(s > 0.0)) { ret = (int)(j + 1); break; }
    const double d = sqrt(s);
    E(A, j, j, lda) = d;
    /* c <- (c - B r^T) / d */
    /* one contiguous row range per thread, m outermost, four terms per pass in the same
     * left-to-right order (see or_chol_fwd_cols) */
    const int64_t rows = n - j - 1;
#pragma omp parallel if (rows * j >= (1 << 16))
    {
      int64_t i0, i1;
      row_range(j + 1, n, &i0, &i1);
      for (int64_t i = i0; i < i1; ++i) t[i] = 0.0;
      int64_t m = 0;
      for (; m + 4 <= j; m += 4) {
        const double r0 = E(A, j, m, lda), r1 = E(A, j, m + 1, lda), r2 = E(A, j, m + 2, lda),
                     r3 = E(A, j, m + 3, lda);
        for (int64_t i = i0; i < i1; ++i) {
          double a = t[i];
          a += E(A, i, m, lda) * r0;
          a += E(A, i, m + 1, lda) * r1;
          a += E(A, i, m + 2, lda) * r2;
          a += E(A, i, m + 3, lda) * r3;
          t[i] = a;
        }
      }
      for (; m < j; ++m) {
        const double r_m = E(A, j, m, lda);
        for (int64_t i = i0; i < i1; ++i) t[i] += E(A, i, m, lda) * r_m;
      }
      for (int64_t i = i0; i < i1; ++i) E(A, i, j, lda) = (E(A, i, j, lda) - t[i]) / d;
    }
  }
  free(t);
  return ret;
}

/* Same algorithm over complex numbers, for complex-step differentiation
 * (an independent pin of the derivative definition; the square root is
 * analytic near the positive reals so Im(chol(Sigma + i h V))/h = Ldot). */
int or_chol_unblocked_complex(int64_t n, double complex* A, int64_t lda) {
  for (int64_t j = 0; j < n; ++j) {
    double complex s = E(A, j, j, lda);
    for (int64_t m = 0; m < j; ++m) s -= E(A, j, m, lda) * E(A, j, m, lda);
    if (!(creal(s) > 0.0)) return (int)(j + 1);
    double complex d = csqrt(s);
    E(A, j, j, lda) = d;
    for (int64_t i = j + 1; i < n; ++i) {
      double complex t = 0.0;
      for (int64_t m = 0; m < j; ++m) t += E(A, i, m, lda) * E(A, j, m, lda);
      E(A, i, j, lda) = (E(A, i, j, lda) - t) / d;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* chol_unblocked_fwd(L, Adot).                             */
/* In place: tril(Adot) = tril(Sigma_dot) -> Ldot.  Returns 0 or j+1 if L_jj  */
/* is zero / non-finite (then the output is unspecified).                     */
/* ------------------------------------------------------------------------- */
int or_chol_fwd(int64_t n, const double* L, int64_t ldl, double* Ad, int64_t lda) {
  for (int64_t j = 0; j < n; ++j) {
    /* r, d, B, c = level2partition(L, j); rdot, ddot, Bdot, cdot = level2partition(Adot, j) */
    double d = E(L, j, j, ldl);
    if (d == 0.0 || !isfinite(d)) return (int)(j + 1);
    /* ddot <- (ddot/2 - r rdot^T) / d */
    double r_rdot = 0.0;
    for (int64_t m = 0; m < j; ++m) r_rdot += E(L, j, m, ldl) * E(Ad, j, m, lda);
    double ddot = (E(Ad, j, j, lda) / 2.0 - r_rdot) / d;
    E(Ad, j, j, lda) = ddot;
    /* cdot <- (cdot - Bdot r^T - B rdot^T - c ddot) / d */
    for (int64_t i = j + 1; i < n; ++i) {
      double Bdot_rT = 0.0, B_rdotT = 0.0;
      for (int64_t m = 0; m < j; ++m) Bdot_rT += E(Ad, i, m, lda) * E(L, j, m, ldl);
      for (int64_t m = 0; m < j; ++m) B_rdotT += E(L, i, m, ldl) * E(Ad, j, m, lda);
      E(Ad, i, j, lda) = (E(Ad, i, j, lda) - Bdot_rT - B_rdotT - E(L, i, j, ldl) * ddot) / d;
    }
  }
  return 0;
}

/* The same statements as or_chol_fwd, evaluated with the  */
/* loop over rows i innermost so that every access walks down a column (the   */
/* column-major layout) -- the only use is large n (full-size parity tests,   */
/* N = 16384), where or_chol_fwd's row-wise walk through a 2 GiB array is     */
/* TLB-bound.  Each sum Bdot r^T, B rdot^T still starts at 0.0 and adds the   */
/* terms m = 0, 1, ..., j-1 in that order, and every other operation is the   */
/* same, so the result is bit-identical to or_chol_fwd (test_oracle.py::      */
/* test_fwd_cols_bit_identical).  Rows i are independent given ddot: OpenMP   */
/* over row ranges.  t1/t2: caller-free scratch of n doubles each.            */
int or_chol_fwd_cols(int64_t n, const double* L, int64_t ldl, double* Ad, int64_t lda) {
  double* t1 = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* t2 = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int ret = 0;
  for (int64_t j = 0; j < n; ++j) {
    double d = E(L, j, j, ldl);
    if (d == 0.0 || !isfinite(d)) { ret = (int)(j + 1); break; }
    /* ddot <- (ddot/2 - r rdot^T) / d */
    double r_rdot = 0.0;
    for (int64_t m = 0; m < j; ++m) r_rdot += E(L, j, m, ldl) * E(Ad, j, m, lda);
    const double ddot = (E(Ad, j, j, lda) / 2.0 - r_rdot) / d;
    E(Ad, j, j, lda) = ddot;
    /* cdot <- (cdot - Bdot r^T - B rdot^T - c ddot) / d */
    /* rows j+1..n-1 split into one contiguous range per thread; within a range the m loop
     * is outermost (column walks) and the per-row sums t1, t2 stay in cache.  Four terms per
     * pass: t = ((t + a_m r_m) + a_{m+1} r_{m+1}) + ...  -- the same left-to-right order. */
    const int64_t rows = n - j - 1;
#pragma omp parallel if (rows * j >= (1 << 16))
    {
      int64_t i0, i1;
      row_range(j + 1, n, &i0, &i1);
      for (int64_t i = i0; i < i1; ++i) { t1[i] = 0.0; t2[i] = 0.0; }
      int64_t m = 0;
      for (; m + 4 <= j; m += 4) {
        const double r0 = E(L, j, m, ldl), r1 = E(L, j, m + 1, ldl), r2 = E(L, j, m + 2, ldl),
                     r3 = E(L, j, m + 3, ldl);
        const double q0 = E(Ad, j, m, lda), q1 = E(Ad, j, m + 1, lda), q2 = E(Ad, j, m + 2, lda),
                     q3 = E(Ad, j, m + 3, lda);
        for (int64_t i = i0; i < i1; ++i) {
          double a = t1[i], b = t2[i];
          a += E(Ad, i, m, lda) * r0;     /* Bdot r^T  */
          a += E(Ad, i, m + 1, lda) * r1;
          a += E(Ad, i, m + 2, lda) * r2;
          a += E(Ad, i, m + 3, lda) * r3;
          b += E(L, i, m, ldl) * q0;      /* B rdot^T  */
          b += E(L, i, m + 1, ldl) * q1;
          b += E(L, i, m + 2, ldl) * q2;
          b += E(L, i, m + 3, ldl) * q3;
          t1[i] = a;
          t2[i] = b;
        }
      }
      for (; m < j; ++m) {
        const double r_m = E(L, j, m, ldl), rdot_m = E(Ad, j, m, lda);
        for (int64_t i = i0; i < i1; ++i) {
          t1[i] += E(Ad, i, m, lda) * r_m;
          t2[i] += E(L, i, m, ldl) * rdot_m;
        }
      }
      for (int64_t i = i0; i < i1; ++i)
        E(Ad, i, j, lda) = (E(Ad, i, j, lda) - t1[i] - t2[i] - E(L, i, j, ldl) * ddot) / d;
    }
  }
  free(t1);
  free(t2);
  return ret;
}

/* ------------------------------------------------------------------------- */
/* chol_unblocked_rev(L, Abar).                             */
/* In place: tril(Abar) = Lbar -> tril(Sigma_bar).  Loop j = N..1.            */
/* Statement order exactly as printed: dbar uses the undivided    */
/* cbar; rbar uses dbar divided by d but not yet halved; halving is last.     */
/* Columns [j_lo, n) only are processed when j_lo > 0 (a bounded sample of    */
/* the sweep, used by bench.py's cpu_baseline; j_lo = 0 is the full sweep).   */
/* ------------------------------------------------------------------------- */
static int rev_sweep(int64_t n, const double* L, int64_t ldl, double* Ab, int64_t lda,
                     int64_t j_lo) {
  for (int64_t j = n - 1; j >= j_lo; --j) {
    double d = E(L, j, j, ldl);
    if (d == 0.0 || !isfinite(d)) return (int)(j + 1);
    /* dbar <- dbar - c^T cbar / d */
    double c_cbar = 0.0;
    for (int64_t i = j + 1; i < n; ++i) c_cbar += E(L, i, j, ldl) * E(Ab, i, j, lda);
    E(Ab, j, j, lda) = E(Ab, j, j, lda) - c_cbar / d;
    /* [dbar; cbar] <- [dbar; cbar] / d */
    E(Ab, j, j, lda) = E(Ab, j, j, lda) / d;
    for (int64_t i = j + 1; i < n; ++i) E(Ab, i, j, lda) = E(Ab, i, j, lda) / d;
    /* rbar <- rbar - [dbar cbar^T] [r; B] */
    /* Bbar <- Bbar - cbar r */
    /* (columns m < j are independent: OpenMP over m for large sweeps) */
    const double dbar = E(Ab, j, j, lda);
#pragma omp parallel for schedule(static) if (j >= 512)
    for (int64_t m = 0; m < j; ++m) {
      double s = dbar * E(L, j, m, ldl);
      for (int64_t i = j + 1; i < n; ++i) s += E(Ab, i, j, lda) * E(L, i, m, ldl);
      E(Ab, j, m, lda) = E(Ab, j, m, lda) - s;
      const double r_m = E(L, j, m, ldl);
      for (int64_t i = j + 1; i < n; ++i) E(Ab, i, m, lda) = E(Ab, i, m, lda) - E(Ab, i, j, lda) * r_m;
    }
    /* dbar <- dbar / 2 */
    E(Ab, j, j, lda) = E(Ab, j, j, lda) / 2.0;
  }
  return 0;
}

int or_chol_rev(int64_t n, const double* L, int64_t ldl, double* Ab, int64_t lda) {
  return rev_sweep(n, L, ldl, Ab, lda, 0);
}

/* Columns j_lo..n-1 of the reverse sweep only (bench sample; see rev_sweep). */
int or_chol_rev_partial(int64_t n, const double* L, int64_t ldl, double* Ab, int64_t lda,
                        int64_t j_lo) {
  return rev_sweep(n, L, ldl, Ab, lda, j_lo);
}

/* Batched drivers (contiguous base + stride); OpenMP over independent matrices.
 * info[b] receives each matrix's return code. */
void or_chol_rev_batched(int64_t n, int64_t batch, const double* L, int64_t ldl, int64_t sL,
                         double* Ab, int64_t lda, int64_t sA, int* info) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    info[b] = or_chol_rev(n, L + b * sL, ldl, Ab + b * sA, lda);
}

void or_chol_fwd_batched(int64_t n, int64_t batch, const double* L, int64_t ldl, int64_t sL,
                         double* Ad, int64_t lda, int64_t sA, int* info) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    info[b] = or_chol_fwd(n, L + b * sL, ldl, Ad + b * sA, lda);
}

/* As or_chol_fwd_batched with the column-ordered evaluation (bit-identical, see
 * or_chol_fwd_cols; its inner OpenMP region stays serial inside this one). */
void or_chol_fwd_cols_batched(int64_t n, int64_t batch, const double* L, int64_t ldl, int64_t sL,
                              double* Ad, int64_t lda, int64_t sA, int* info) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t b = 0; b < batch; ++b)
    info[b] = or_chol_fwd_cols(n, L + b * sL, ldl, Ad + b * sA, lda);
}

/* ------------------------------------------------------------------------- */
/* Second, independent oracle: the symbolic results of Section 3, evaluated   */
/* with plain forward / back substitution (no explicit inverse is formed).    */
/* All work arrays are dense n x n, column-major, ld = n.                     */
/* ------------------------------------------------------------------------- */

/* Phi (Eq. 6): lower triangle with the diagonal halved. */
static void phi_inplace(int64_t n, double* X) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      if (i < j) E(X, i, j, n) = 0.0;
      else if (i == j) E(X, i, j, n) = E(X, i, j, n) / 2.0;
    }
}

/* Solve L X = B in place (B <- L^{-1} B), L lower, forward substitution. */
static void solve_L(int64_t n, const double* L, int64_t ldl, double* B) {
  for (int64_t c = 0; c < n; ++c)
    for (int64_t i = 0; i < n; ++i) {
      double t = E(B, i, c, n);
      for (int64_t m = 0; m < i; ++m) t -= E(L, i, m, ldl) * E(B, m, c, n);
      E(B, i, c, n) = t / E(L, i, i, ldl);
    }
}

/* Solve L^T X = B in place (B <- L^{-T} B), back substitution. */
static void solve_LT(int64_t n, const double* L, int64_t ldl, double* B) {
  for (int64_t c = 0; c < n; ++c)
    for (int64_t i = n - 1; i >= 0; --i) {
      double t = E(B, i, c, n);
      for (int64_t m = i + 1; m < n; ++m) t -= E(L, m, i, ldl) * E(B, m, c, n);
      E(B, i, c, n) = t / E(L, i, i, ldl);
    }
}

static void transpose(int64_t n, const double* X, double* Y) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) E(Y, i, j, n) = E(X, j, i, n);
}

static int diag_ok(int64_t n, const double* L, int64_t ldl) {
  for (int64_t j = 0; j < n; ++j) {
    double d = E(L, j, j, ldl);
    if (d == 0.0 || !isfinite(d)) return (int)(j + 1);
  }
  return 0;
}

/* Eq. 8: Ldot = L Phi(L^{-1} Sdot L^{-T}).
 * Sdot is read from tril(Sd) and mirrored (Sdot symmetric).
 * Output: Ldot written to the lower triangle of Out (ld = ldo), upper = 0. */
int or_chol_fwd_symbolic(int64_t n, const double* L, int64_t ldl, const double* Sd, int64_t lds,
                         double* Out, int64_t ldo) {
  int bad = diag_ok(n, L, ldl);
  if (bad || n == 0) return bad;
  double* X = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * n * n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) E(X, i, j, n) = (i >= j) ? E(Sd, i, j, lds) : E(Sd, j, i, lds);
  solve_L(n, L, ldl, X);          /* X = L^{-1} Sdot                    */
  transpose(n, X, Y);             /* Y = (L^{-1} Sdot)^T = Sdot L^{-T}  */
  solve_L(n, L, ldl, Y);          /* Y = L^{-1} Sdot L^{-T}             */
  phi_inplace(n, Y);              /* Phi(...)                           */
  for (int64_t j = 0; j < n; ++j) /* Out = L Phi(...)                   */
    for (int64_t i = 0; i < n; ++i) {
      double t = 0.0;
      for (int64_t m = 0; m < n; ++m) {
        double l = (i >= m) ? E(L, i, m, ldl) : 0.0;
        t += l * E(Y, m, j, n);
      }
      E(Out, i, j, ldo) = t;
    }
  free(X);
  free(Y);
  return 0;
}

/* P = Phi(L^T Lbar), dense n x n output. */
static void make_P(int64_t n, const double* L, int64_t ldl, const double* Lb, int64_t ldb,
                   double* P) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double t = 0.0;
      for (int64_t m = 0; m < n; ++m) {
        double lmi = (m >= i) ? E(L, m, i, ldl) : 0.0;   /* (L^T)_{i m} = L_{m i} */
        double bmj = (m >= j) ? E(Lb, m, j, ldb) : 0.0;  /* tril(Lbar)_{m j}      */
        t += lmi * bmj;
      }
      E(P, i, j, n) = t;
    }
  phi_inplace(n, P);
}

/* Eq. 10: tril(Sbar) = Phi(L^{-T} (P + P^T) L^{-1}).
 * Output in the lower triangle of Out, upper triangle set to 0. */
int or_chol_rev_symbolic(int64_t n, const double* L, int64_t ldl, const double* Lb, int64_t ldb,
                         double* Out, int64_t ldo) {
  int bad = diag_ok(n, L, ldl);
  if (bad || n == 0) return bad;
  double* P = (double*)malloc(sizeof(double) * n * n);
  double* X = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * n * n);
  make_P(n, L, ldl, Lb, ldb, P);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) E(X, i, j, n) = E(P, i, j, n) + E(P, j, i, n); /* P + P^T */
  solve_LT(n, L, ldl, X);         /* X = L^{-T} (P + P^T)                          */
  transpose(n, X, Y);             /* Y = X^T                                       */
  solve_LT(n, L, ldl, Y);         /* Y = L^{-T} X^T = (X L^{-1})^T                 */
  transpose(n, Y, X);             /* X = L^{-T} (P + P^T) L^{-1}                   */
  phi_inplace(n, X);              /* Phi(...)                                      */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) E(Out, i, j, ldo) = E(X, i, j, n);
  free(P);
  free(X);
  free(Y);
  return 0;
}

/* Eq. 9: Sbar = S + S^T - diag(S), S = L^{-T} Phi(L^T Lbar) L^{-1}.
 * Full symmetric output in Out. */
int or_chol_rev_symbolic_sym(int64_t n, const double* L, int64_t ldl, const double* Lb,
                             int64_t ldb, double* Out, int64_t ldo) {
  int bad = diag_ok(n, L, ldl);
  if (bad || n == 0) return bad;
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * n * n);
  make_P(n, L, ldl, Lb, ldb, S);  /* S = P                                          */
  solve_LT(n, L, ldl, S);         /* S = L^{-T} P                                   */
  transpose(n, S, Y);             /* Y = P^T L^{-1}                                 */
  solve_LT(n, L, ldl, Y);         /* Y = L^{-T} P^T L^{-1} = S^T                    */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      /* S_{ij} = Y_{ji};  Sbar_{ij} = S_{ij} + S_{ji} - [i==j] S_{ii} */
      double sij = E(Y, j, i, n), sji = E(Y, i, j, n);
      E(Out, i, j, ldo) = (i == j) ? sij : sij + sji;
    }
  free(S);
  free(Y);
  return 0;
}
