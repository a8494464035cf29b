/*
 * h2oracle.c — CPU restatement of the reference h2cross hot path
 * (tree build, neighbour / interaction lists, partially pivoted ACA,
 * NNCA pivot selection with interpolation operators, H2 matvec).
 *
 * TEST INFRASTRUCTURE ONLY (see h2oracle.h).  The product library
 * (paper_2203_14832_b200/csrc) never links or calls this code.
 *
 * Floating-point contract: compiled with -ffp-contract=off so every
 * expression rounds exactly as the reference's Cython core (_core.pyx,
 * built with plain -O3, no FMA) does.  The one place the reference goes
 * through OpenBLAS (np.dot in geometry.py:152) is restated with explicit
 * fma() in sequence, which is what that ddot kernel computes for d <= 8
 * (checked against numpy in tests/test_oracle_golden.py).
 */
#include "h2oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXD 8
#define WIDTH_UNDERFLOW 0x1p-50 /* geometry.py:36 */
#define TOP_COMPRESSED_LEVEL 2  /* compress.py:40 */
static const double INV_FOUR_PI = 0.07957747154594767; /* 1/(4 pi), correctly rounded */

static char g_err[512];
const char* oh2_last_error(void) { return g_err; }
static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

static int g_threads = 0;
void oh2_set_threads(int n) { g_threads = n; }
int oh2_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "h2oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "h2oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------ */
/* kernels: _core.pyx:15 _kval, :38 _r2                              */
/* ------------------------------------------------------------------ */
double oh2_kval(int kind, double a, double r2) {
  double r;
  if (kind == OH2_GAUSSIAN) return exp(-r2);
  if (kind == OH2_GAUSSIAN_SCALED) return exp(-(a * r2));
  r = sqrt(r2);
  switch (kind) {
    case OH2_MATERN:
      return exp(-r);
    case OH2_COULOMB:
      return r == 0.0 ? 0.0 : 1.0 / r;
    case OH2_LAPLACE:
      return r == 0.0 ? 0.0 : INV_FOUR_PI / r;
    case OH2_LOG:
      return r == 0.0 ? 0.0 : log(r);
    case OH2_REG_INVERSE:
      return r < a ? r / a : a / r;
    default: /* OH2_REG_LOG */
      if (r >= a) return log(r) / log(a);
      if (r == 0.0) return 0.0;
      return (r * (log(r) - 1.0)) / (a * (log(a) - 1.0));
  }
}

static inline double r2_of(const double* x, const double* y, int d) {
  double acc = 0.0, diff;
  for (int k = 0; k < d; k++) {
    diff = x[k] - y[k];
    acc += diff * diff;
  }
  return acc;
}

void oh2_kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n,
                      int d, double* out) {
  for (int64_t i = 0; i < m; i++)
    for (int64_t j = 0; j < n; j++) out[i * n + j] = oh2_kval(kind, a, r2_of(X + i * d, Y + j * d, d));
}

/* ------------------------------------------------------------------ */
/* geometry: geometry.py:147 boxes_admissible                          */
/* ------------------------------------------------------------------ */
int oh2_boxes_admissible(const double* cx, double hwx, const double* cy, double hwy, int d,
                         double eta) {
  double diam = 2.0 * (hwx > hwy ? hwx : hwy) * sqrt((double)d);
  double dot = 0.0;
  for (int k = 0; k < d; k++) {
    double g = fabs(cx[k] - cy[k]) - (hwx + hwy);
    g = g > 0.0 ? g : 0.0; /* np.maximum(., 0.0) */
    dot = fma(g, g, dot);  /* OpenBLAS ddot: sequential fused accumulation */
  }
  double dist = sqrt(dot);
  return diam <= eta * dist;
}

/* ------------------------------------------------------------------ */
/* tree                                                                */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t *key, *mi;
  int64_t *t_ptr, *t_idx, *s_ptr, *s_idx;
  int64_t *parent, *ch_ptr, *ch_idx;
  int64_t *nb_ptr, *nb_idx, *il_ptr, *il_idx;
  double* center;
  double hw;
  int over_cap;
} olevel;

struct oh2_tree {
  int d, shared, depth, over_capacity;
  int64_t np, nq, nu;
  double eta, half, mid[MAXD], lo0[MAXD];
  double *P, *Q; /* copies (row-major) */
  olevel* lv;
};

typedef struct {
  int64_t key, idx;
} kpair;
static int cmp_kpair(const void* a, const void* b) {
  const kpair* x = (const kpair*)a;
  const kpair* y = (const kpair*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static int64_t find_key(const int64_t* keys, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == key) ? lo : -1;
}

static int64_t ravel(const int64_t* mi, int d, int level) {
  int64_t k = 0;
  for (int j = 0; j < d; j++) k = (k << level) | mi[j];
  return k;
}

static void level_free(olevel* L) {
  free(L->key); free(L->mi); free(L->t_ptr); free(L->t_idx); free(L->s_ptr); free(L->s_idx);
  free(L->parent); free(L->ch_ptr); free(L->ch_idx); free(L->nb_ptr); free(L->nb_idx);
  free(L->il_ptr); free(L->il_idx); free(L->center);
}

void oh2_tree_free(oh2_tree* t) {
  if (!t) return;
  for (int l = 0; l <= t->depth; l++) {
    olevel* L = &t->lv[l];
    if (L->s_idx == L->t_idx) L->s_idx = NULL;
    if (L->s_ptr == L->t_ptr) L->s_ptr = NULL;
    level_free(L);
  }
  free(t->lv);
  if (t->Q != t->P) free(t->Q);
  free(t->P);
  free(t);
}

/* sort a small list of cell indices by their level keys (insertion sort:
 * lists are at most a few hundred entries) — geometry.py:333-334 */
static void sort_by_key(int64_t* idx, int64_t n, const int64_t* keys) {
  for (int64_t i = 1; i < n; i++) {
    int64_t v = idx[i], kv = keys[v], j = i - 1;
    while (j >= 0 && keys[idx[j]] > kv) {
      idx[j + 1] = idx[j];
      j--;
    }
    idx[j + 1] = v;
  }
}

/* geometry.py:322 _annotate_level restricted to nonempty cells (empty cells
 * have no points and no nonempty descendants, so they never contribute to
 * any candidate set, coupling or near-field block) */
static void annotate_level(oh2_tree* t, int level) {
  olevel* L = &t->lv[level];
  olevel* Lp = &t->lv[level - 1];
  int d = t->d;
  int64_t n = L->n;
  int64_t* nb_cnt = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
  int64_t* il_cnt = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
  /* pass 1: counts */
#pragma omp parallel for schedule(dynamic, 64) num_threads(oh2_get_threads())
  for (int64_t b = 0; b < n; b++) {
    int64_t p = L->parent[b], cn = 0, ci = 0;
    for (int64_t q = Lp->nb_ptr[p]; q < Lp->nb_ptr[p + 1]; q++) {
      int64_t nb = Lp->nb_idx[q];
      for (int64_t r = Lp->ch_ptr[nb]; r < Lp->ch_ptr[nb + 1]; r++) {
        int64_t c = Lp->ch_idx[r];
        if (oh2_boxes_admissible(L->center + b * d, L->hw, L->center + c * d, L->hw, d, t->eta)) ci++;
        else cn++;
      }
    }
    nb_cnt[b + 1] = cn;
    il_cnt[b + 1] = ci;
  }
  for (int64_t b = 0; b < n; b++) {
    nb_cnt[b + 1] += nb_cnt[b];
    il_cnt[b + 1] += il_cnt[b];
  }
  L->nb_ptr = nb_cnt;
  L->il_ptr = il_cnt;
  L->nb_idx = (int64_t*)xmalloc(sizeof(int64_t) * nb_cnt[n]);
  L->il_idx = (int64_t*)xmalloc(sizeof(int64_t) * il_cnt[n]);
#pragma omp parallel for schedule(dynamic, 64) num_threads(oh2_get_threads())
  for (int64_t b = 0; b < n; b++) {
    int64_t p = L->parent[b], wn = L->nb_ptr[b], wi = L->il_ptr[b];
    for (int64_t q = Lp->nb_ptr[p]; q < Lp->nb_ptr[p + 1]; q++) {
      int64_t nb = Lp->nb_idx[q];
      for (int64_t r = Lp->ch_ptr[nb]; r < Lp->ch_ptr[nb + 1]; r++) {
        int64_t c = Lp->ch_idx[r];
        if (oh2_boxes_admissible(L->center + b * d, L->hw, L->center + c * d, L->hw, d, t->eta))
          L->il_idx[wi++] = c;
        else
          L->nb_idx[wn++] = c;
      }
    }
    sort_by_key(L->nb_idx + L->nb_ptr[b], L->nb_ptr[b + 1] - L->nb_ptr[b], L->key);
    sort_by_key(L->il_idx + L->il_ptr[b], L->il_ptr[b + 1] - L->il_ptr[b], L->key);
  }
}

/* group (key, idx) pairs (sorted) -> per-cell ranges, for the cells list */
static void fill_ranges(const kpair* pr, int64_t npts, const int64_t* keys, int64_t ncell,
                        int64_t** ptr_out, int64_t** idx_out) {
  int64_t* ptr = (int64_t*)xcalloc(ncell + 1, sizeof(int64_t));
  int64_t* idx = (int64_t*)xmalloc(sizeof(int64_t) * npts);
  int64_t c = 0;
  for (int64_t i = 0; i < npts; i++) {
    while (keys[c] != pr[i].key) c++;
    ptr[c + 1]++;
    idx[i] = pr[i].idx;
  }
  for (int64_t k = 0; k < ncell; k++) ptr[k + 1] += ptr[k];
  *ptr_out = ptr;
  *idx_out = idx;
}

int oh2_build_tree(const double* P, int64_t np, const double* Q, int64_t nq, int d, int shared,
                   int64_t nu, double eta, oh2_tree** out) {
  /* geometry.py:235-240 */
  if (np == 0 || nq == 0) return fail("empty point set");
  if (nu < 1) return fail("invalid leaf capacity");
  if (!(eta > 0)) return fail("eta must be positive");
  if (d < 1 || d > MAXD) return fail("dimension %d unsupported (1..%d)", d, MAXD);
  if (shared && np != nq) return fail("shared cloud needs equal point counts");

  oh2_tree* t = (oh2_tree*)xcalloc(1, sizeof(oh2_tree));
  t->d = d;
  t->shared = shared;
  t->np = np;
  t->nq = nq;
  t->nu = nu;
  t->eta = eta;
  t->P = (double*)xmalloc(sizeof(double) * np * d);
  memcpy(t->P, P, sizeof(double) * np * d);
  if (shared) t->Q = t->P;
  else {
    t->Q = (double*)xmalloc(sizeof(double) * nq * d);
    memcpy(t->Q, Q, sizeof(double) * nq * d);
  }

  /* geometry.py:243-247 root box */
  double lo[MAXD], hi[MAXD];
  for (int k = 0; k < d; k++) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (int64_t i = 0; i < np; i++)
    for (int k = 0; k < d; k++) {
      double v = t->P[i * d + k];
      if (v < lo[k]) lo[k] = v;
      if (v > hi[k]) hi[k] = v;
    }
  if (!shared)
    for (int64_t i = 0; i < nq; i++)
      for (int k = 0; k < d; k++) {
        double v = t->Q[i * d + k];
        if (v < lo[k]) lo[k] = v;
        if (v > hi[k]) hi[k] = v;
      }
  double hm = -INFINITY;
  for (int k = 0; k < d; k++) {
    t->mid[k] = 0.5 * (lo[k] + hi[k]);
    double e = hi[k] - t->mid[k];
    if (e > hm) hm = e;
  }
  double half = hm > 0 ? hm : 1.0;
  half *= 1.0 + 1e-12;
  t->half = half;
  for (int k = 0; k < d; k++) t->lo0[k] = t->mid[k] - half;

  int cap_levels = 64;
  t->lv = (olevel*)xcalloc(cap_levels, sizeof(olevel));
  /* level 0: the root */
  olevel* R = &t->lv[0];
  R->n = 1;
  R->key = (int64_t*)xcalloc(1, sizeof(int64_t));
  R->mi = (int64_t*)xcalloc(d, sizeof(int64_t));
  R->center = (double*)xmalloc(sizeof(double) * d);
  for (int k = 0; k < d; k++) R->center[k] = t->mid[k];
  R->hw = half;
  R->t_ptr = (int64_t*)xmalloc(2 * sizeof(int64_t));
  R->t_ptr[0] = 0;
  R->t_ptr[1] = np;
  R->t_idx = (int64_t*)xmalloc(sizeof(int64_t) * np);
  for (int64_t i = 0; i < np; i++) R->t_idx[i] = i;
  if (shared) {
    R->s_ptr = R->t_ptr;
    R->s_idx = R->t_idx;
  } else {
    R->s_ptr = (int64_t*)xmalloc(2 * sizeof(int64_t));
    R->s_ptr[0] = 0;
    R->s_ptr[1] = nq;
    R->s_idx = (int64_t*)xmalloc(sizeof(int64_t) * nq);
    for (int64_t i = 0; i < nq; i++) R->s_idx[i] = i;
  }
  R->parent = (int64_t*)xcalloc(1, sizeof(int64_t));
  R->parent[0] = -1;
  R->nb_ptr = (int64_t*)xmalloc(2 * sizeof(int64_t));
  R->nb_ptr[0] = 0;
  R->nb_ptr[1] = 1;
  R->nb_idx = (int64_t*)xcalloc(1, sizeof(int64_t)); /* root is its own neighbour */
  R->il_ptr = (int64_t*)xcalloc(2, sizeof(int64_t));
  R->il_idx = (int64_t*)xcalloc(1, sizeof(int64_t));

  int64_t* bins_p = (int64_t*)xcalloc(np * d, sizeof(int64_t));
  int64_t* bins_q = shared ? bins_p : (int64_t*)xcalloc(nq * d, sizeof(int64_t));
  int level = 0;
  int rc = 0;
  for (;;) {
    /* geometry.py:264-267 */
    olevel* L = &t->lv[level];
    int64_t worst = 0;
    for (int64_t c = 0; c < L->n; c++) {
      int64_t a = L->t_ptr[c + 1] - L->t_ptr[c], b = L->s_ptr[c + 1] - L->s_ptr[c];
      int64_t w = a > b ? a : b;
      if (w > worst) worst = w;
    }
    if (worst <= nu) break;
    /* geometry.py:268-273 */
    double width = half * ldexp(1.0, -level);
    if (width / (2.0 * half) < WIDTH_UNDERFLOW) {
      for (int64_t c = 0; c < L->n; c++) {
        int64_t a = L->t_ptr[c + 1] - L->t_ptr[c], b = L->s_ptr[c + 1] - L->s_ptr[c];
        if ((a > b ? a : b) > nu) L->over_cap = 1;
      }
      t->over_capacity = 1;
      break;
    }
    if ((int64_t)(level + 1) * d >= 63) {
      /* np.ravel_multi_index overflow in geometry.py:303 */
      rc = fail("invalid dims: array size defined by dims is larger than the maximum possible size.");
      break;
    }
    /* geometry.py:275-279 bin refinement, exact reference arithmetic */
    double w2 = 2.0 * width;
    for (int pass = 0; pass < (shared ? 1 : 2); pass++) {
      const double* pts = pass == 0 ? t->P : t->Q;
      int64_t* bins = pass == 0 ? bins_p : bins_q;
      int64_t n = pass == 0 ? np : nq;
#pragma omp parallel for schedule(static) num_threads(oh2_get_threads())
      for (int64_t i = 0; i < n; i++)
        for (int k = 0; k < d; k++) {
          double c = t->lo0[k] + ((double)bins[i * d + k] + 0.5) * w2;
          bins[i * d + k] = 2 * bins[i * d + k] + (pts[i * d + k] > c ? 1 : 0);
        }
    }
    level++;
    if (level >= cap_levels) {
      rc = fail("tree too deep");
      break;
    }
    /* geometry.py:302-311 grouping */
    kpair* pp = (kpair*)xmalloc(sizeof(kpair) * np);
    for (int64_t i = 0; i < np; i++) {
      pp[i].key = ravel(bins_p + i * d, d, level);
      pp[i].idx = i;
    }
    qsort(pp, np, sizeof(kpair), cmp_kpair);
    kpair* pq = pp;
    if (!shared) {
      pq = (kpair*)xmalloc(sizeof(kpair) * nq);
      for (int64_t i = 0; i < nq; i++) {
        pq[i].key = ravel(bins_q + i * d, d, level);
        pq[i].idx = i;
      }
      qsort(pq, nq, sizeof(kpair), cmp_kpair);
    }
    /* union of occupied keys (nonempty cells), ascending */
    int64_t* keys = (int64_t*)xmalloc(sizeof(int64_t) * (np + (shared ? 0 : nq)));
    int64_t nk = 0, i = 0, j = 0;
    int64_t nqq = shared ? 0 : nq;
    while (i < np || j < nqq) {
      int64_t k;
      if (j >= nqq || (i < np && pp[i].key <= pq[j].key)) k = pp[i].key;
      else k = pq[j].key;
      if (nk == 0 || keys[nk - 1] != k) keys[nk++] = k;
      while (i < np && pp[i].key == k) i++;
      while (j < nqq && pq[j].key == k) j++;
    }
    olevel* N = &t->lv[level];
    N->n = nk;
    N->key = keys;
    N->mi = (int64_t*)xmalloc(sizeof(int64_t) * nk * d);
    N->center = (double*)xmalloc(sizeof(double) * nk * d);
    double wl = half * ldexp(1.0, 1 - level); /* cell width at this level */
    N->hw = 0.5 * wl;
    for (int64_t c = 0; c < nk; c++) {
      int64_t k = keys[c];
      for (int q = d - 1; q >= 0; q--) {
        N->mi[c * d + q] = k & ((1LL << level) - 1);
        k >>= level;
      }
      for (int q = 0; q < d; q++)
        N->center[c * d + q] = t->lo0[q] + ((double)N->mi[c * d + q] + 0.5) * wl;
    }
    fill_ranges(pp, np, keys, nk, &N->t_ptr, &N->t_idx);
    if (shared) {
      N->s_ptr = N->t_ptr;
      N->s_idx = N->t_idx;
    } else {
      fill_ranges(pq, nq, keys, nk, &N->s_ptr, &N->s_idx);
      free(pq);
    }
    free(pp);
    /* parent / children links */
    olevel* Lp = &t->lv[level - 1];
    N->parent = (int64_t*)xmalloc(sizeof(int64_t) * nk);
    int64_t pmi[MAXD];
    for (int64_t c = 0; c < nk; c++) {
      for (int q = 0; q < d; q++) pmi[q] = N->mi[c * d + q] >> 1;
      N->parent[c] = find_key(Lp->key, Lp->n, ravel(pmi, d, level - 1));
    }
    Lp->ch_ptr = (int64_t*)xcalloc(Lp->n + 1, sizeof(int64_t));
    for (int64_t c = 0; c < nk; c++) Lp->ch_ptr[N->parent[c] + 1]++;
    for (int64_t c = 0; c < Lp->n; c++) Lp->ch_ptr[c + 1] += Lp->ch_ptr[c];
    Lp->ch_idx = (int64_t*)xmalloc(sizeof(int64_t) * (nk ? nk : 1));
    {
      int64_t* fillp = (int64_t*)xmalloc(sizeof(int64_t) * (Lp->n + 1));
      memcpy(fillp, Lp->ch_ptr, sizeof(int64_t) * (Lp->n + 1));
      for (int64_t c = 0; c < nk; c++) Lp->ch_idx[fillp[N->parent[c]]++] = c; /* key order */
      free(fillp);
    }
    annotate_level(t, level);
  }
  t->depth = level;
  /* leaves have no children */
  olevel* Lf = &t->lv[level];
  Lf->ch_ptr = (int64_t*)xcalloc(Lf->n + 1, sizeof(int64_t));
  Lf->ch_idx = (int64_t*)xcalloc(1, sizeof(int64_t));
  free(bins_p);
  if (!shared) free(bins_q);
  if (rc) {
    oh2_tree_free(t);
    return rc;
  }
  *out = t;
  return 0;
}

int oh2_tree_depth(const oh2_tree* t) { return t->depth; }
int oh2_tree_over_capacity(const oh2_tree* t) { return t->over_capacity; }
void oh2_tree_root(const oh2_tree* t, double* mid, double* half) {
  for (int k = 0; k < t->d; k++) mid[k] = t->mid[k];
  *half = t->half;
}
int64_t oh2_tree_ncells(const oh2_tree* t, int level) { return t->lv[level].n; }

int64_t oh2_tree_get(const oh2_tree* t, int level, int what, int64_t* dst) {
  const olevel* L = &t->lv[level];
  const int64_t* src = NULL;
  int64_t n = 0;
  switch (what) {
    case 0: src = L->key; n = L->n; break;
    case 1: src = L->mi; n = L->n * t->d; break;
    case 2: src = L->t_ptr; n = L->n + 1; break;
    case 3: src = L->t_idx; n = L->t_ptr[L->n]; break;
    case 4: src = L->s_ptr; n = L->n + 1; break;
    case 5: src = L->s_idx; n = L->s_ptr[L->n]; break;
    case 6: src = L->nb_ptr; n = L->n + 1; break;
    case 7: src = L->nb_idx; n = L->nb_ptr[L->n]; break;
    case 8: src = L->il_ptr; n = L->n + 1; break;
    case 9: src = L->il_idx; n = L->il_ptr[L->n]; break;
    case 10: src = L->parent; n = L->n; break;
    case 11: src = L->ch_ptr; n = L->n + 1; break;
    case 12: src = L->ch_idx; n = L->ch_ptr[L->n]; break;
    default: return -1;
  }
  if (dst && n) memcpy(dst, src, sizeof(int64_t) * n);
  return n;
}

/* ------------------------------------------------------------------ */
/* ACA: _core.pyx:70 aca_kernel                                       */
/* U, V kept column-major by rank (U[t*m+i], V[t*n+j]); the arithmetic  */
/* order per entry is exactly the reference's.                         */
/* ------------------------------------------------------------------ */
typedef struct {
  double *U, *V;
  int64_t *rp, *cp;
  int64_t k, nevals;
  int converged;
} acares;

static void aca_core(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n,
                     int d, double eps, int64_t cap, acares* res) {
  int64_t full = m < n ? m : n;
  int64_t alloc = cap < 32 ? cap : 32;
  double* U = (double*)xmalloc(sizeof(double) * m * alloc);
  double* V = (double*)xmalloc(sizeof(double) * n * alloc);
  int64_t* rp = (int64_t*)xmalloc(sizeof(int64_t) * cap);
  int64_t* cp = (int64_t*)xmalloc(sizeof(int64_t) * cap);
  unsigned char* row_used = (unsigned char*)xcalloc(m, 1);
  unsigned char* col_used = (unsigned char*)xcalloc(n, 1);
  double* urow = (double*)xmalloc(sizeof(double) * cap);
  double* vrow = (double*)xmalloc(sizeof(double) * cap);
  int64_t k = 0, trial = 0, nevals = 0;
  double norm2 = 0.0;
  int converged = 1, exhausted = 0;

  for (;;) {
    if (k == alloc) { /* grow: same contents, more rank columns */
      alloc = alloc * 2 < cap ? alloc * 2 : cap;
      U = (double*)realloc(U, sizeof(double) * m * alloc);
      V = (double*)realloc(V, sizeof(double) * n * alloc);
      if (!U || !V) abort();
    }
    int64_t best_j = -1;
    double best;
    for (;;) {
      best = -1.0;
      best_j = -1;
      row_used[trial] = 1;
      for (int64_t t = 0; t < k; t++) urow[t] = U[t * m + trial];
      const double* xt = X + trial * d;
      double* Vk = V + k * n;
      for (int64_t j = 0; j < n; j++) {
        double acc = oh2_kval(kind, a, r2_of(xt, Y + j * d, d));
        for (int64_t t = 0; t < k; t++) acc -= urow[t] * V[t * n + j];
        Vk[j] = acc;
        if (!col_used[j]) {
          double val = fabs(acc);
          if (val > best) {
            best = val;
            best_j = j;
          }
        }
      }
      nevals += n;
      if (best > 0.0) break;
      exhausted = 1;
      for (int64_t i = 0; i < m; i++)
        if (!row_used[i]) {
          trial = i;
          exhausted = 0;
          break;
        }
      if (exhausted) break;
    }
    if (exhausted) break;

    int64_t j = best_j;
    double* Vk = V + k * n;
    double piv = Vk[j];
    for (int64_t t = 0; t < n; t++) Vk[t] /= piv;
    col_used[j] = 1;
    for (int64_t t = 0; t < k; t++) vrow[t] = V[t * n + j];
    const double* yj = Y + j * d;
    double* Uk = U + k * m;
    for (int64_t i = 0; i < m; i++) {
      double acc = oh2_kval(kind, a, r2_of(X + i * d, yj, d));
      for (int64_t t = 0; t < k; t++) acc -= U[t * m + i] * vrow[t];
      Uk[i] = acc;
    }
    nevals += m;
    rp[k] = trial;
    cp[k] = j;

    double u2 = 0.0, v2 = 0.0;
    for (int64_t i = 0; i < m; i++) u2 += Uk[i] * Uk[i];
    for (int64_t t = 0; t < n; t++) v2 += Vk[t] * Vk[t];
    for (int64_t t = 0; t < k; t++) {
      double cross = 0.0, acc = 0.0;
      const double* Ut = U + t * m;
      const double* Vt = V + t * n;
      for (int64_t i = 0; i < m; i++) cross += Ut[i] * Uk[i];
      for (int64_t i = 0; i < n; i++) acc += Vt[i] * Vk[i];
      norm2 += 2.0 * cross * acc;
    }
    norm2 += u2 * v2;
    k += 1;

    if (u2 * v2 <= eps * eps * (norm2 > 0.0 ? norm2 : 0.0)) break;
    if (k == full) break;
    if (k == cap) {
      converged = 0;
      break;
    }
    best = -1.0;
    int64_t best_i = -1;
    for (int64_t i = 0; i < m; i++)
      if (!row_used[i]) {
        double val = fabs(Uk[i]);
        if (val > best) {
          best = val;
          best_i = i;
        }
      }
    if (best_i < 0) break;
    trial = best_i;
  }
  free(row_used);
  free(col_used);
  free(urow);
  free(vrow);
  res->U = U;
  res->V = V;
  res->rp = rp;
  res->cp = cp;
  res->k = k;
  res->nevals = nevals;
  res->converged = converged;
}

int64_t oh2_aca(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d,
                double eps, int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp,
                int* converged, int64_t* nevals) {
  if (m == 0 || n == 0 || cap == 0) {
    *converged = (m == 0 || n == 0) ? 1 : 0;
    *nevals = 0;
    return 0;
  }
  acares r;
  aca_core(kind, a, X, m, Y, n, d, eps, cap, &r);
  for (int64_t i = 0; i < m; i++)
    for (int64_t t = 0; t < r.k; t++) U[i * cap + t] = r.U[t * m + i];
  for (int64_t j = 0; j < n; j++)
    for (int64_t t = 0; t < r.k; t++) V[j * cap + t] = r.V[t * n + j];
  memcpy(rp, r.rp, sizeof(int64_t) * r.k);
  memcpy(cp, r.cp, sizeof(int64_t) * r.k);
  *converged = r.converged;
  *nevals = r.nevals;
  free(r.U); free(r.V); free(r.rp); free(r.cp);
  return r.k;
}

/* aca.py:297 row_interpolator: P = U L^{-1}, L = tril(U[rp]); P[rp] = I.
 * Uc column-major (Uc[t*m+i]); out row-major (m x k). */
static void row_interp_cm(const double* Uc, int64_t m, int64_t k, const int64_t* rp, double* out) {
  for (int64_t i = 0; i < m; i++) {
    double* p = out + i * k;
    for (int64_t s = k - 1; s >= 0; s--) {
      double acc = Uc[s * m + i];
      for (int64_t t = s + 1; t < k; t++) acc -= p[t] * Uc[s * m + rp[t]];
      p[s] = acc / Uc[s * m + rp[s]];
    }
  }
  for (int64_t t = 0; t < k; t++) {
    double* p = out + rp[t] * k;
    for (int64_t s = 0; s < k; s++) p[s] = (s == t) ? 1.0 : 0.0;
  }
}

/* aca.py:311 col_interpolator: Q = V R^{-T}, R = triu(V[cp].T), unit diag;
 * Q[cp] = I.  Vc column-major; out row-major (n x k). */
static void col_interp_cm(const double* Vc, int64_t n, int64_t k, const int64_t* cp, double* out) {
  for (int64_t j = 0; j < n; j++) {
    double* q = out + j * k;
    for (int64_t s = k - 1; s >= 0; s--) {
      double acc = Vc[s * n + j];
      for (int64_t t = s + 1; t < k; t++) acc -= q[t] * Vc[s * n + cp[t]];
      q[s] = acc;
    }
  }
  for (int64_t t = 0; t < k; t++) {
    double* q = out + cp[t] * k;
    for (int64_t s = 0; s < k; s++) q[s] = (s == t) ? 1.0 : 0.0;
  }
}

void oh2_row_interpolator(const double* U, int64_t m, int64_t k, const int64_t* rp, double* out) {
  double* Uc = (double*)xmalloc(sizeof(double) * m * k);
  for (int64_t i = 0; i < m; i++)
    for (int64_t t = 0; t < k; t++) Uc[t * m + i] = U[i * k + t];
  row_interp_cm(Uc, m, k, rp, out);
  free(Uc);
}

void oh2_col_interpolator(const double* V, int64_t n, int64_t k, const int64_t* cp, double* out) {
  double* Vc = (double*)xmalloc(sizeof(double) * n * k);
  for (int64_t j = 0; j < n; j++)
    for (int64_t t = 0; t < k; t++) Vc[t * n + j] = V[j * k + t];
  col_interp_cm(Vc, n, k, cp, out);
  free(Vc);
}

/* ------------------------------------------------------------------ */
/* NNCA: compress.py:159 candidate_sets, :216 select_pivots, :285       */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t *kin, *kout;                 /* per cell */
  int64_t *in_ptr, *out_ptr;           /* scans of kin / kout */
  int64_t *t_in, *s_in, *t_out, *s_out; /* global pivot indices */
  int64_t *nevals;
  int64_t* conv_in;
  double** interp; /* row interp (m_in x kin) row-major */
  double** anterp; /* col interp (n_out x kout); == interp when symmetric */
  int64_t *m_in, *n_out;
} ohlevel;

struct oh2_h2 {
  const oh2_tree* t;
  int kind, symmetric;
  double a;
  ohlevel* lv; /* indexed by level; only levels >= 2 populated */
  int64_t evals_pivots, evals_couplings, evals_nearfield, max_rank, cells_visited;
};

static void gather_pts(const double* pts, const int64_t* idx, int64_t n, int d, double* out) {
  for (int64_t i = 0; i < n; i++) memcpy(out + i * d, pts + idx[i] * d, sizeof(double) * d);
}

void oh2_h2_free(oh2_h2* h) {
  if (!h) return;
  for (int l = TOP_COMPRESSED_LEVEL; l <= h->t->depth; l++) {
    ohlevel* H = &h->lv[l];
    for (int64_t c = 0; c < H->n; c++) {
      if (H->anterp[c] != H->interp[c]) free(H->anterp[c]);
      free(H->interp[c]);
    }
    free(H->interp); free(H->anterp); free(H->kin); free(H->kout); free(H->in_ptr);
    free(H->out_ptr); free(H->t_in); free(H->s_in); free(H->t_out); free(H->s_out);
    free(H->nevals); free(H->conv_in); free(H->m_in); free(H->n_out);
  }
  free(h->lv);
  free(h);
}

/* per-cell candidate lists (compress.py:159-209) */
static int64_t* cand_list(const oh2_tree* t, const oh2_h2* h, int level, int64_t b, int which,
                          int64_t* count) {
  /* which: 0 t_in, 1 s_in, 2 t_out, 3 s_out */
  const olevel* L = &t->lv[level];
  int leaf = level == t->depth;
  int64_t n = 0, *out;
  if (leaf) {
    if (which == 0 || which == 3) {
      const int64_t* ptr = which == 0 ? L->t_ptr : L->s_ptr;
      const int64_t* idx = which == 0 ? L->t_idx : L->s_idx;
      n = ptr[b + 1] - ptr[b];
      out = (int64_t*)xmalloc(sizeof(int64_t) * (n ? n : 1));
      memcpy(out, idx + ptr[b], sizeof(int64_t) * n);
    } else {
      const int64_t* ptr = which == 1 ? L->s_ptr : L->t_ptr;
      const int64_t* idx = which == 1 ? L->s_idx : L->t_idx;
      for (int64_t q = L->il_ptr[b]; q < L->il_ptr[b + 1]; q++) {
        int64_t c = L->il_idx[q];
        n += ptr[c + 1] - ptr[c];
      }
      out = (int64_t*)xmalloc(sizeof(int64_t) * (n ? n : 1));
      int64_t w = 0;
      for (int64_t q = L->il_ptr[b]; q < L->il_ptr[b + 1]; q++) {
        int64_t c = L->il_idx[q];
        memcpy(out + w, idx + ptr[c], sizeof(int64_t) * (ptr[c + 1] - ptr[c]));
        w += ptr[c + 1] - ptr[c];
      }
    }
  } else {
    const ohlevel* C = &h->lv[level + 1];
    /* which 0: children t_in; 3: children s_out; 1: IL children s_out; 2: IL children t_in */
    const int64_t* cptr = (which == 0 || which == 2) ? C->in_ptr : C->out_ptr;
    const int64_t* cidx = (which == 0 || which == 2) ? C->t_in : C->s_out;
    int64_t nmem = (which == 0 || which == 3) ? 1 : L->il_ptr[b + 1] - L->il_ptr[b];
    for (int pass = 0; pass < 2; pass++) {
      int64_t w = 0;
      for (int64_t q = 0; q < nmem; q++) {
        int64_t mem = (which == 0 || which == 3) ? b : L->il_idx[L->il_ptr[b] + q];
        for (int64_t r = L->ch_ptr[mem]; r < L->ch_ptr[mem + 1]; r++) {
          int64_t ch = L->ch_idx[r];
          int64_t len = cptr[ch + 1] - cptr[ch];
          if (pass) memcpy(out + w, cidx + cptr[ch], sizeof(int64_t) * len);
          w += len;
        }
      }
      if (!pass) {
        n = w;
        out = (int64_t*)xmalloc(sizeof(int64_t) * (n ? n : 1));
      }
    }
  }
  *count = n;
  return out;
}

int oh2_assemble(const oh2_tree* t, int kind, double a, double eps, int force_general,
                 int64_t max_rank, oh2_h2** out) {
  if (!(eps > 0)) return fail("epsilon must be positive");
  oh2_h2* h = (oh2_h2*)xcalloc(1, sizeof(oh2_h2));
  h->t = t;
  h->kind = kind;
  h->a = a;
  h->symmetric = t->shared && !force_general; /* all built-in kernels are symmetric */
  h->lv = (ohlevel*)xcalloc(t->depth + 1, sizeof(ohlevel));
  int d = t->d;
  for (int level = t->depth; level >= TOP_COMPRESSED_LEVEL; level--) {
    const olevel* L = &t->lv[level];
    ohlevel* H = &h->lv[level];
    int64_t n = L->n;
    H->n = n;
    H->kin = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->kout = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->nevals = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->conv_in = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->m_in = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->n_out = (int64_t*)xcalloc(n, sizeof(int64_t));
    H->interp = (double**)xcalloc(n, sizeof(double*));
    H->anterp = (double**)xcalloc(n, sizeof(double*));
    int64_t** tin = (int64_t**)xcalloc(n, sizeof(int64_t*));
    int64_t** sin = (int64_t**)xcalloc(n, sizeof(int64_t*));
    int64_t** tout = (int64_t**)xcalloc(n, sizeof(int64_t*));
    int64_t** sout = (int64_t**)xcalloc(n, sizeof(int64_t*));
#pragma omp parallel for schedule(dynamic, 1) num_threads(oh2_get_threads())
    for (int64_t b = 0; b < n; b++) {
      int64_t m, nn;
      int64_t* rows = cand_list(t, h, level, b, 0, &m);
      int64_t* cols = cand_list(t, h, level, b, 1, &nn);
      double* X = (double*)xmalloc(sizeof(double) * (m ? m : 1) * d);
      double* Y = (double*)xmalloc(sizeof(double) * (nn ? nn : 1) * d);
      gather_pts(t->P, rows, m, d, X);
      gather_pts(t->Q, cols, nn, d, Y);
      int64_t cap = m < nn ? m : nn;
      if (max_rank >= 0 && max_rank < cap) cap = max_rank;
      acares r;
      memset(&r, 0, sizeof r);
      r.converged = 1;
      if (m > 0 && nn > 0) {
        if (cap > 0) aca_core(kind, a, X, m, Y, nn, d, eps, cap, &r);
        else r.converged = 0;
      }
      int64_t k = r.k;
      H->kin[b] = k;
      H->nevals[b] = r.nevals;
      H->conv_in[b] = r.converged;
      H->m_in[b] = m;
      tin[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k ? k : 1));
      sin[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k ? k : 1));
      for (int64_t q = 0; q < k; q++) {
        tin[b][q] = rows[r.rp[q]];
        sin[b][q] = cols[r.cp[q]];
      }
      H->interp[b] = (double*)xmalloc(sizeof(double) * (m * k > 0 ? m * k : 1));
      if (k) row_interp_cm(r.U, m, k, r.rp, H->interp[b]);
      free(r.U); free(r.V); free(r.rp); free(r.cp);
      free(X); free(Y); free(rows); free(cols);
      if (h->symmetric) {
        H->kout[b] = k;
        H->n_out[b] = m;
        tout[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k ? k : 1));
        sout[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k ? k : 1));
        memcpy(tout[b], sin[b], sizeof(int64_t) * k);
        memcpy(sout[b], tin[b], sizeof(int64_t) * k);
        H->anterp[b] = H->interp[b];
      } else {
        int64_t mo, no;
        int64_t* rows2 = cand_list(t, h, level, b, 2, &mo);
        int64_t* cols2 = cand_list(t, h, level, b, 3, &no);
        double* X2 = (double*)xmalloc(sizeof(double) * (mo ? mo : 1) * d);
        double* Y2 = (double*)xmalloc(sizeof(double) * (no ? no : 1) * d);
        gather_pts(t->P, rows2, mo, d, X2);
        gather_pts(t->Q, cols2, no, d, Y2);
        int64_t cap2 = mo < no ? mo : no;
        if (max_rank >= 0 && max_rank < cap2) cap2 = max_rank;
        acares r2;
        memset(&r2, 0, sizeof r2);
        if (mo > 0 && no > 0 && cap2 > 0) aca_core(kind, a, X2, mo, Y2, no, d, eps, cap2, &r2);
        int64_t k2 = r2.k;
        H->kout[b] = k2;
        H->nevals[b] += r2.nevals;
        H->n_out[b] = no;
        tout[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k2 ? k2 : 1));
        sout[b] = (int64_t*)xmalloc(sizeof(int64_t) * (k2 ? k2 : 1));
        for (int64_t q = 0; q < k2; q++) {
          tout[b][q] = rows2[r2.rp[q]];
          sout[b][q] = cols2[r2.cp[q]];
        }
        H->anterp[b] = (double*)xmalloc(sizeof(double) * (no * k2 > 0 ? no * k2 : 1));
        if (k2) col_interp_cm(r2.V, no, k2, r2.cp, H->anterp[b]);
        free(r2.U); free(r2.V); free(r2.rp); free(r2.cp);
        free(X2); free(Y2); free(rows2); free(cols2);
      }
    }
    /* compact pivots into per-level CSR */
    H->in_ptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
    H->out_ptr = (int64_t*)xcalloc(n + 1, sizeof(int64_t));
    for (int64_t b = 0; b < n; b++) {
      H->in_ptr[b + 1] = H->in_ptr[b] + H->kin[b];
      H->out_ptr[b + 1] = H->out_ptr[b] + H->kout[b];
      h->evals_pivots += H->nevals[b];
      h->cells_visited++;
      if (H->kin[b] > h->max_rank) h->max_rank = H->kin[b];
      if (H->kout[b] > h->max_rank) h->max_rank = H->kout[b];
    }
    H->t_in = (int64_t*)xmalloc(sizeof(int64_t) * (H->in_ptr[n] ? H->in_ptr[n] : 1));
    H->s_in = (int64_t*)xmalloc(sizeof(int64_t) * (H->in_ptr[n] ? H->in_ptr[n] : 1));
    H->t_out = (int64_t*)xmalloc(sizeof(int64_t) * (H->out_ptr[n] ? H->out_ptr[n] : 1));
    H->s_out = (int64_t*)xmalloc(sizeof(int64_t) * (H->out_ptr[n] ? H->out_ptr[n] : 1));
    for (int64_t b = 0; b < n; b++) {
      memcpy(H->t_in + H->in_ptr[b], tin[b], sizeof(int64_t) * H->kin[b]);
      memcpy(H->s_in + H->in_ptr[b], sin[b], sizeof(int64_t) * H->kin[b]);
      memcpy(H->t_out + H->out_ptr[b], tout[b], sizeof(int64_t) * H->kout[b]);
      memcpy(H->s_out + H->out_ptr[b], sout[b], sizeof(int64_t) * H->kout[b]);
      free(tin[b]); free(sin[b]); free(tout[b]); free(sout[b]);
    }
    free(tin); free(sin); free(tout); free(sout);
  }
  /* compress.py:307-328 entry counts of couplings and near field */
  for (int level = TOP_COMPRESSED_LEVEL; level <= t->depth; level++) {
    const olevel* L = &t->lv[level];
    const ohlevel* H = &h->lv[level];
    for (int64_t b = 0; b < L->n; b++) {
      if (!H->kin[b]) continue;
      for (int64_t q = L->il_ptr[b]; q < L->il_ptr[b + 1]; q++)
        h->evals_couplings += H->kin[b] * H->kout[L->il_idx[q]];
    }
  }
  {
    const olevel* L = &t->lv[t->depth];
    for (int64_t b = 0; b < L->n; b++) {
      int64_t nt = L->t_ptr[b + 1] - L->t_ptr[b];
      for (int64_t q = L->nb_ptr[b]; q < L->nb_ptr[b + 1]; q++) {
        int64_t c = L->nb_idx[q];
        h->evals_nearfield += nt * (L->s_ptr[c + 1] - L->s_ptr[c]);
      }
    }
  }
  *out = h;
  return 0;
}

int64_t oh2_h2_get_i64(const oh2_h2* h, int level, int what, int64_t* dst) {
  const ohlevel* H = &h->lv[level];
  const int64_t* src = NULL;
  int64_t n = 0;
  if (level < TOP_COMPRESSED_LEVEL || level > h->t->depth) return 0;
  switch (what) {
    case 0: src = H->kin; n = H->n; break;
    case 1: src = H->kout; n = H->n; break;
    case 2: src = H->t_in; n = H->in_ptr[H->n]; break;
    case 3: src = H->s_in; n = H->in_ptr[H->n]; break;
    case 4: src = H->t_out; n = H->out_ptr[H->n]; break;
    case 5: src = H->s_out; n = H->out_ptr[H->n]; break;
    case 6: src = H->nevals; n = H->n; break;
    case 7: src = H->conv_in; n = H->n; break;
    default: return -1;
  }
  if (dst && n) memcpy(dst, src, sizeof(int64_t) * n);
  return n;
}

int64_t oh2_h2_get_interp(const oh2_h2* h, int level, int64_t cell, int which, int64_t* cols,
                          double* dst) {
  const ohlevel* H = &h->lv[level];
  int64_t rows = which == 0 ? H->m_in[cell] : H->n_out[cell];
  int64_t k = which == 0 ? H->kin[cell] : H->kout[cell];
  if (cols) *cols = k;
  if (dst && rows * k > 0) memcpy(dst, which == 0 ? H->interp[cell] : H->anterp[cell], sizeof(double) * rows * k);
  return rows;
}

void oh2_h2_stats(const oh2_h2* h, int64_t* evals_pivots, int64_t* evals_couplings,
                  int64_t* evals_nearfield, int64_t* max_rank, int64_t* cells_visited) {
  *evals_pivots = h->evals_pivots;
  *evals_couplings = h->evals_couplings;
  *evals_nearfield = h->evals_nearfield;
  *max_rank = h->max_rank;
  *cells_visited = h->cells_visited;
}

/* ------------------------------------------------------------------ */
/* matvec: matvec.py:169 h2_matvec_reference (S and near-field blocks   */
/* regenerated entry by entry instead of stored)                        */
/* ------------------------------------------------------------------ */
int oh2_matvec(const oh2_h2* h, const double* w, double* u, int64_t nrhs) {
  const oh2_tree* t = h->t;
  int d = t->d, depth = t->depth;
  int64_t R = nrhs;
  memset(u, 0, sizeof(double) * t->np * R);
  double** wout = (double**)xcalloc(depth + 1, sizeof(double*));
  double** uin = (double**)xcalloc(depth + 1, sizeof(double*));
  if (depth >= TOP_COMPRESSED_LEVEL) {
    for (int l = TOP_COMPRESSED_LEVEL; l <= depth; l++) {
      const ohlevel* H = &h->lv[l];
      wout[l] = (double*)xcalloc(H->out_ptr[H->n] * R + 1, sizeof(double));
      uin[l] = (double*)xcalloc(H->in_ptr[H->n] * R + 1, sizeof(double));
    }
    /* upward pass: leaf P2M, then M2M */
    {
      const olevel* L = &t->lv[depth];
      const ohlevel* H = &h->lv[depth];
#pragma omp parallel for schedule(dynamic, 16) num_threads(oh2_get_threads())
      for (int64_t b = 0; b < L->n; b++) {
        int64_t k = H->kout[b], ns = L->s_ptr[b + 1] - L->s_ptr[b];
        const double* Qm = H->anterp[b]; /* ns x k */
        double* wo = wout[depth] + H->out_ptr[b] * R;
        for (int64_t s = 0; s < k; s++)
          for (int64_t rr = 0; rr < R; rr++) {
            double acc = 0.0;
            for (int64_t j = 0; j < ns; j++) acc += Qm[j * k + s] * w[L->s_idx[L->s_ptr[b] + j] * R + rr];
            wo[s * R + rr] = acc;
          }
      }
    }
    for (int l = depth - 1; l >= TOP_COMPRESSED_LEVEL; l--) {
      const olevel* L = &t->lv[l];
      const ohlevel* H = &h->lv[l];
      const ohlevel* C = &h->lv[l + 1];
#pragma omp parallel for schedule(dynamic, 16) num_threads(oh2_get_threads())
      for (int64_t b = 0; b < L->n; b++) {
        int64_t k = H->kout[b];
        const double* Qm = H->anterp[b];
        double* wo = wout[l] + H->out_ptr[b] * R;
        int64_t row = 0;
        for (int64_t r = L->ch_ptr[b]; r < L->ch_ptr[b + 1]; r++) {
          int64_t ch = L->ch_idx[r];
          const double* wc = wout[l + 1] + C->out_ptr[ch] * R;
          for (int64_t j = 0; j < C->kout[ch]; j++, row++)
            for (int64_t s = 0; s < k; s++)
              for (int64_t rr = 0; rr < R; rr++) wo[s * R + rr] += Qm[row * k + s] * wc[j * R + rr];
        }
      }
    }
    /* transverse pass: u_in(B) = sum_{B' in IL(B)} K(t_in^B, s_out^B') w_out(B') */
    for (int l = TOP_COMPRESSED_LEVEL; l <= depth; l++) {
      const olevel* L = &t->lv[l];
      const ohlevel* H = &h->lv[l];
#pragma omp parallel for schedule(dynamic, 4) num_threads(oh2_get_threads())
      for (int64_t b = 0; b < L->n; b++) {
        double* ui = uin[l] + H->in_ptr[b] * R;
        for (int64_t a = 0; a < H->kin[b]; a++) {
          const double* x = t->P + H->t_in[H->in_ptr[b] + a] * d;
          for (int64_t q = L->il_ptr[b]; q < L->il_ptr[b + 1]; q++) {
            int64_t c = L->il_idx[q];
            const double* wo = wout[l] + H->out_ptr[c] * R;
            for (int64_t s = 0; s < H->kout[c]; s++) {
              double kv = oh2_kval(h->kind, h->a, r2_of(x, t->Q + H->s_out[H->out_ptr[c] + s] * d, d));
              for (int64_t rr = 0; rr < R; rr++) ui[a * R + rr] += kv * wo[s * R + rr];
            }
          }
        }
      }
    }
    /* downward pass */
    for (int l = TOP_COMPRESSED_LEVEL; l < depth; l++) {
      const olevel* L = &t->lv[l];
      const ohlevel* H = &h->lv[l];
      const ohlevel* C = &h->lv[l + 1];
#pragma omp parallel for schedule(dynamic, 16) num_threads(oh2_get_threads())
      for (int64_t b = 0; b < L->n; b++) {
        int64_t k = H->kin[b];
        const double* Pm = H->interp[b];
        const double* ui = uin[l] + H->in_ptr[b] * R;
        int64_t row = 0;
        for (int64_t r = L->ch_ptr[b]; r < L->ch_ptr[b + 1]; r++) {
          int64_t ch = L->ch_idx[r];
          double* uc = uin[l + 1] + C->in_ptr[ch] * R;
          for (int64_t i = 0; i < C->kin[ch]; i++, row++)
            for (int64_t rr = 0; rr < R; rr++) {
              double acc = 0.0;
              for (int64_t s = 0; s < k; s++) acc += Pm[row * k + s] * ui[s * R + rr];
              uc[i * R + rr] += acc;
            }
        }
      }
    }
    /* leaf L2P */
    {
      const olevel* L = &t->lv[depth];
      const ohlevel* H = &h->lv[depth];
#pragma omp parallel for schedule(dynamic, 16) num_threads(oh2_get_threads())
      for (int64_t b = 0; b < L->n; b++) {
        int64_t k = H->kin[b], nt = L->t_ptr[b + 1] - L->t_ptr[b];
        const double* Pm = H->interp[b];
        const double* ui = uin[depth] + H->in_ptr[b] * R;
        for (int64_t i = 0; i < nt; i++)
          for (int64_t rr = 0; rr < R; rr++) {
            double acc = 0.0;
            for (int64_t s = 0; s < k; s++) acc += Pm[i * k + s] * ui[s * R + rr];
            u[L->t_idx[L->t_ptr[b] + i] * R + rr] += acc;
          }
      }
    }
  }
  /* near field (matvec.py:220-226) */
  {
    const olevel* L = &t->lv[depth];
#pragma omp parallel for schedule(dynamic, 16) num_threads(oh2_get_threads())
    for (int64_t b = 0; b < L->n; b++) {
      for (int64_t i = L->t_ptr[b]; i < L->t_ptr[b + 1]; i++) {
        int64_t ti = L->t_idx[i];
        const double* x = t->P + ti * d;
        for (int64_t q = L->nb_ptr[b]; q < L->nb_ptr[b + 1]; q++) {
          int64_t c = L->nb_idx[q];
          for (int64_t j = L->s_ptr[c]; j < L->s_ptr[c + 1]; j++) {
            int64_t sj = L->s_idx[j];
            double kv = oh2_kval(h->kind, h->a, r2_of(x, t->Q + sj * d, d));
            for (int64_t rr = 0; rr < R; rr++) u[ti * R + rr] += kv * w[sj * R + rr];
          }
        }
      }
    }
  }
  for (int l = 0; l <= depth; l++) {
    free(wout[l]);
    free(uin[l]);
  }
  free(wout);
  free(uin);
  return 0;
}

void oh2_dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq,
                      int d, const double* w, double* u, int64_t nrhs) {
#pragma omp parallel for schedule(static) num_threads(oh2_get_threads())
  for (int64_t i = 0; i < np; i++) {
    for (int64_t rr = 0; rr < nrhs; rr++) u[i * nrhs + rr] = 0.0;
    for (int64_t j = 0; j < nq; j++) {
      double kv = oh2_kval(kind, a, r2_of(P + i * d, Q + j * d, d));
      for (int64_t rr = 0; rr < nrhs; rr++) u[i * nrhs + rr] += kv * w[j * nrhs + rr];
    }
  }
}

void oh2_dense_rows(int kind, double a, const double* P, const int64_t* rows, int64_t nrows,
                    const double* Q, int64_t nq, int d, const double* w, double* u) {
#pragma omp parallel for schedule(static) num_threads(oh2_get_threads())
  for (int64_t r = 0; r < nrows; r++) {
    double acc = 0.0;
    const double* x = P + rows[r] * d;
    for (int64_t j = 0; j < nq; j++) acc += oh2_kval(kind, a, r2_of(x, Q + j * d, d)) * w[j];
    u[r] = acc;
  }
}
