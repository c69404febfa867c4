/*
 * ebc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C fp64 restatement of the reference hot path (ebcsum 0.1.0,
 * /root/reference/pkg/src/ebcsum).  It is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library (libebc200.so)
 * never links or calls anything in this directory.
 *
 * Semantics followed (reference file:line):
 *   - squared Euclidean distance, exact direct-difference form, fp64
 *       core.py:205-217 (squared_euclidean), core.py:278-293 (cross)
 *   - loss L(S u {e0}) = ordered fp64 sum over v of min_{r in {e0} u S} d(v,r), / N
 *       ebc.py:13-18 (_ordered_sum), ebc.py:74-88 (loss_of_indices)
 *   - baseline L({e0}) computed once            ebc.py:72
 *   - f(S) = baseline - L(S u {e0})             ebc.py:90-92
 *   - multiset evaluation, values in set order, IndexError naming the set
 *       ebc.py:109-121, core.py:136-143
 *   - Greedy: full frontier each step, argmax with tie window
 *     1e-12*max(1,|top|) and lowest index, gains = value - previous,
 *     evaluations += |frontier|                  optimize.py:60-91
 *
 * The Greedy restatement uses the cached-min identity
 *     min_{r in {e0} u S u {c}} d(v,r) = min(cm_S(v), d(v,c)),
 * with cm_S kept in fp64; min is exact, so every candidate value is the same
 * fp64 expression the reference's naive backend evaluates, without the O(|S|)
 * rescan.  Per-candidate sums are sequential over v (ascending), so results do
 * not depend on the OpenMP thread count.
 *
 * Return codes: 0 ok, 1 invalid argument, 2 index error (out_bad_set /
 * out_bad_index say which), matching the C-ABI convention of include/ebc200.h.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* d(x, y) = sum_k (x_k - y_k)^2, ascending k, fp64 (core.py:216-217). */
static inline double sqdist(const double* x, const double* y, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = x[k] - y[k];
    s += t * t;
  }
  return s;
}


/* Tiled copy of V: groups of 16 consecutive points stored as [k][16], so the
 * distance loop reads 128 contiguous bytes per dimension.  Each point's sum is
 * still sequential over k, so values are bit-identical to sqdist(); only
 * independent points are computed side by side.  Rows past n are zero. */
#define TG 32
static double* transpose(const double* V, int64_t n, int d) {
  const int64_t ng = (n + TG - 1) / TG;
  double* VT = (double*)calloc((size_t)ng * TG * (size_t)d, sizeof(double));
  if (!VT) return NULL;
  for (int64_t v = 0; v < n; ++v)
    for (int k = 0; k < d; ++k) VT[(size_t)(v / TG) * d * TG + (size_t)k * TG + (v % TG)] = V[v * d + k];
  return VT;
}

#define OB 512 /* points per block (multiple of TG) */

/* out[i] = d(V[v0+i], y) for i < nb (v0 a multiple of TG).  GCC vector
 * extensions keep 16 per-point accumulators in registers; lanes are points,
 * so every point's sum stays sequential over k. */
typedef double v8d __attribute__((vector_size(64)));
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
__attribute__((target_clones("avx512f", "avx2", "default")))
#endif
static void dist_block(const double* __restrict VT, int64_t n, int d, int64_t v0, int nb,
                       const double* __restrict y, double* __restrict out) {
  (void)n;
  for (int i = 0; i < nb; i += TG) {
    const double* __restrict g = VT + (size_t)((v0 + i) / TG) * d * TG;
    v8d a0 = {0, 0, 0, 0, 0, 0, 0, 0}, a1 = a0, a2 = a0, a3 = a0;
    for (int k = 0; k < d; ++k) {
      v8d x0, x1, x2, x3;
      memcpy(&x0, g + k * TG, sizeof(x0));
      memcpy(&x1, g + k * TG + 8, sizeof(x1));
      memcpy(&x2, g + k * TG + 16, sizeof(x2));
      memcpy(&x3, g + k * TG + 24, sizeof(x3));
      const double yk = y[k];
      v8d t0 = x0 - yk, t1 = x1 - yk, t2 = x2 - yk, t3 = x3 - yk;
      a0 = a0 + t0 * t0;
      a1 = a1 + t1 * t1;
      a2 = a2 + t2 * t2;
      a3 = a3 + t3 * t3;
    }
    double acc[TG];
    memcpy(acc, &a0, sizeof(a0));
    memcpy(acc + 8, &a1, sizeof(a1));
    memcpy(acc + 16, &a2, sizeof(a2));
    memcpy(acc + 24, &a3, sizeof(a3));
    const int m = nb - i < TG ? nb - i : TG;
    for (int j = 0; j < m; ++j) out[i + j] = acc[j];
  }
}

double ebc_oracle_sqdist(const double* x, const double* y, int d) { return sqdist(x, y, d); }

int ebc_oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ebc_oracle_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* e0d[v] = d(v, e0); baseline = ordered_sum(e0d) / n  (ebc.py:72,74-88). */
int ebc_oracle_baseline(const double* V, int64_t n, int d, const double* e0, double* out_e0d,
                        double* out_baseline) {
  if (!V || !e0 || n < 1 || d < 1) return 1;
  double total = 0.0;
  for (int64_t v = 0; v < n; ++v) {
    double t = sqdist(V + v * d, e0, d);
    if (out_e0d) out_e0d[v] = t;
    total += t;
  }
  if (out_baseline) *out_baseline = total / (double)n;
  return 0;
}

/* f_j = baseline - L(S_j u {e0}) for CSR sets (ebc.py:109-121). */
int ebc_oracle_eval_multiset(const double* V, int64_t n, int d, const double* e0,
                             const int64_t* offsets, const int64_t* idx, int64_t l,
                             double* out, int64_t* out_bad_set, int64_t* out_bad_index) {
  if (!V || !e0 || !offsets || !out || n < 1 || d < 1 || l < 1) return 1;
  /* index validation first, in set order (core.py:136-143) */
  for (int64_t j = 0; j < l; ++j) {
    for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p) {
      if (idx[p] < 0 || idx[p] >= n) {
        if (out_bad_set) *out_bad_set = j;
        if (out_bad_index) *out_bad_index = idx[p];
        return 2;
      }
    }
  }
  double* e0d = (double*)malloc(sizeof(double) * (size_t)n);
  double* VT = transpose(V, n, d);
  if (!e0d || !VT) { free(e0d); free(VT); return 1; }
  double baseline = 0.0;
  ebc_oracle_baseline(V, n, d, e0, e0d, &baseline);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < l; ++j) {
    double m[OB], t[OB];
    double total = 0.0;
    for (int64_t v0 = 0; v0 < n; v0 += OB) {
      int nb = (int)((n - v0) < OB ? (n - v0) : OB);
      for (int i = 0; i < nb; ++i) m[i] = e0d[v0 + i];
      for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p) {
        dist_block(VT, n, d, v0, nb, V + idx[p] * d, t);
        for (int i = 0; i < nb; ++i) m[i] = t[i] < m[i] ? t[i] : m[i];
      }
      for (int i = 0; i < nb; ++i) total += m[i]; /* ordered over v */
    }
    out[j] = baseline - total / (double)n;
  }
  free(e0d);
  free(VT);
  return 0;
}

/* values[c] = baseline - ordered_sum_v min(cm[v], d(v,c)) / n for the listed
 * candidates.  Point blocks are the outer loop so a block stays cache-resident
 * while every candidate consumes it; each candidate's running total still adds
 * its terms strictly left to right over v (ebc.py:13-18). */
static void candidate_values(const double* V, const double* VT, int64_t n, int d, const double* cm,
                             double baseline, const int64_t* cand, int64_t ncand, double* out) {
  double* tot = (double*)calloc((size_t)(ncand > 0 ? ncand : 1), sizeof(double));
  for (int64_t v0 = 0; v0 < n; v0 += OB) {
    const int nb = (int)((n - v0) < OB ? (n - v0) : OB);
    /* 4 candidates per task: their running totals are independent chains */
    const int64_t ngrp = (ncand + 3) / 4;
#pragma omp parallel for schedule(static)
    for (int64_t gi = 0; gi < ngrp; ++gi) {
      double t[4][OB];
      const int64_t i0 = gi * 4;
      const int m = (int)((ncand - i0) < 4 ? (ncand - i0) : 4);
      for (int a = 0; a < m; ++a) dist_block(VT, n, d, v0, nb, V + cand[i0 + a] * d, t[a]);
      if (m == 4) {
        double s0 = tot[i0], s1 = tot[i0 + 1], s2 = tot[i0 + 2], s3 = tot[i0 + 3];
        for (int q = 0; q < nb; ++q) {
          const double c = cm[v0 + q];
          s0 += c < t[0][q] ? c : t[0][q];
          s1 += c < t[1][q] ? c : t[1][q];
          s2 += c < t[2][q] ? c : t[2][q];
          s3 += c < t[3][q] ? c : t[3][q];
        }
        tot[i0] = s0; tot[i0 + 1] = s1; tot[i0 + 2] = s2; tot[i0 + 3] = s3;
      } else {
        for (int a = 0; a < m; ++a) {
          double s = tot[i0 + a];
          for (int q = 0; q < nb; ++q) s += cm[v0 + q] < t[a][q] ? cm[v0 + q] : t[a][q];
          tot[i0 + a] = s;
        }
      }
    }
  }
  for (int64_t i = 0; i < ncand; ++i) out[i] = baseline - tot[i] / (double)n;
  free(tot);
}

static void fold_into_cm(const double* V, const double* VT, int64_t n, int d, int64_t s, double* cm) {
  double t[OB];
  for (int64_t v0 = 0; v0 < n; v0 += OB) {
    int nb = (int)((n - v0) < OB ? (n - v0) : OB);
    dist_block(VT, n, d, v0, nb, V + s * d, t);
    for (int q = 0; q < nb; ++q)
      if (t[q] < cm[v0 + q]) cm[v0 + q] = t[q];
  }
}

/* Greedy (optimize.py:60-91) with the cached-min identity.
 * out_sel/out_val/out_gain hold k entries; out_val[s] = f(S_{s+1}). */
int ebc_oracle_greedy(const double* V, int64_t n, int d, const double* e0, int k,
                      int64_t* out_sel, double* out_val, double* out_gain, int64_t* out_evals) {
  if (!V || !e0 || n < 1 || d < 1 || k < 1 || k > n) return 1;
  double* cm = (double*)malloc(sizeof(double) * (size_t)n);
  double* val = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* remaining = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  double* VT = transpose(V, n, d);
  if (!cm || !val || !remaining || !VT) {
    free(cm); free(val); free(remaining); free(VT);
    return 1;
  }
  double baseline = 0.0;
  ebc_oracle_baseline(V, n, d, e0, cm, &baseline);
  for (int64_t c = 0; c < n; ++c) remaining[c] = c; /* ascending (optimize.py:78) */
  int64_t nrem = n;
  double current = 0.0;
  int64_t evals = 0;
  for (int step = 0; step < k; ++step) {
    candidate_values(V, VT, n, d, cm, baseline, remaining, nrem, val);
    evals += nrem;
    double top = -INFINITY;
    for (int64_t i = 0; i < nrem; ++i)
      if (val[i] > top) top = val[i];
    double window = 1e-12 * (fabs(top) > 1.0 ? fabs(top) : 1.0);
    int64_t bi = 0;
    for (int64_t i = 0; i < nrem; ++i)
      if (val[i] >= top - window) { bi = i; break; }
    int64_t best = remaining[bi];
    out_sel[step] = best;
    out_gain[step] = val[bi] - current;
    current = val[bi];
    out_val[step] = current;
    memmove(remaining + bi, remaining + bi + 1, sizeof(int64_t) * (size_t)(nrem - bi - 1));
    --nrem;
    fold_into_cm(V, VT, n, d, best, cm);
  }
  if (out_evals) *out_evals = evals;
  free(cm); free(val); free(remaining); free(VT);
  return 0;
}

/* Values f(S u {c}) of one Greedy step for the listed candidates, given the
 * selected prefix S: lets the tests audit single steps where a full run is
 * too slow. */
int ebc_oracle_step_values(const double* V, int64_t n, int d, const double* e0,
                           const int64_t* selected, int s, const int64_t* cand, int64_t ncand,
                           double* out_val) {
  if (!V || !e0 || n < 1 || d < 1 || s < 0) return 1;
  double* cm = (double*)malloc(sizeof(double) * (size_t)n);
  double* VT = transpose(V, n, d);
  if (!cm || !VT) { free(cm); free(VT); return 1; }
  double baseline = 0.0;
  ebc_oracle_baseline(V, n, d, e0, cm, &baseline);
  for (int i = 0; i < s; ++i) fold_into_cm(V, VT, n, d, selected[i], cm);
  candidate_values(V, VT, n, d, cm, baseline, cand, ncand, out_val);
  free(cm);
  free(VT);
  return 0;
}

/* k-medoids loss of explicit representatives (ebc.py:21-43): per ground row the
 * minimum over reps of the exact fp64 distance (starting from +inf), summed left
 * to right (_ordered_sum, ebc.py:13-18), divided by n. */
int ebc_oracle_kmedoids(const double* V, int64_t n, int d, const double* reps, int64_t r, double* out) {
  if (!V || !reps || !out || n < 1 || d < 1 || r < 1) return 1;
  double* mins = (double*)malloc((size_t)n * sizeof(double));
  if (!mins) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    double m = INFINITY;
    for (int64_t j = 0; j < r; ++j) {
      const double t = sqdist(V + v * d, reps + j * d, d);
      if (t < m) m = t;
    }
    mins[v] = m;
  }
  double s = 0.0;
  for (int64_t v = 0; v < n; ++v) s += mins[v];
  free(mins);
  *out = s / (double)n;
  return 0;
}
