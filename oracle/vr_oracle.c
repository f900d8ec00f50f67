/*
 * vr_oracle.c — the CPU ORACLE for the Vietoris–Rips barcode (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load or call this file's library.  The product path (paper_2502_05063_b200,
 * libvr.so) shares no code, header, table or helper with it and never calls it.
 *
 * What it computes (SURVEY.md §8(c) "Definition"): the persistence barcode over Z/2 of
 * the Vietoris–Rips filtration of an fp32 distance matrix truncated at a threshold t,
 * for dimensions 0..D, by the textbook route with no shortcut of any kind:
 *
 *   1. enumerate every simplex of dimension 0..D+1 as a vertex subset, diam = max
 *      pairwise distance (Eq 5.3), keep diam <= t (inclusive);
 *   2. order them by the simplex-wise refinement of §5.1.4:
 *      diameter ascending, then dimension ascending, then combinatorial index
 *      DEscending; cidx is Eq 5.6 and is used only for this tie-break and as
 *      the simplex's name in the index-level output;
 *   3. build the Z/2 boundary matrix: column j = the filtration positions of the
 *      facets of simplex j (Def 2.6.7; Fig 4.1);
 *   4. reduce it with the standard algorithm, Alg 2: left to right,
 *      while R[j] != 0 and L[low(R[j])] is set, add that column; then record the pivot.
 *      low() of the zero column is an explicit NONE (reading A17: Eq 3.89 says 0,
 *      Alg 2 says -1; both collide with a real row index);
 *   5. pairs: every pivot (i = low(j), j) is the bar [diam(i), diam(j)) in dimension
 *      dim(i); every simplex i of dim <= D that is neither a pivot row nor a nonzero
 *      column is an essential bar [diam(i), +inf) (Thm 3.2.20).
 *
 * No clearing, no cohomology, no apparent pairs, no implicit matrix.
 *
 * A second entry point, oracle_apparent(), is Def 5.3.4 written out on
 * explicit cofacet / facet sets: (s, t) is apparent iff s is the youngest facet of t
 * and t is the oldest cofacet of s, ages taken in the §5.1.4 order.
 *
 * A third, oracle_reduce_columns(), is Alg 2 alone on a caller-given explicit matrix
 * (used to pin the reduction core on the Fig 4.1 / Fig 4.2 worked example).
 *
 * Pins: tests/test_oracle_pins.py (closed forms, worked examples, persistent Betti
 * numbers by independent rank computations, count identities, brute force).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXV 12 /* at most 12 vertices per simplex (max_dim <= 10) */
#define NONE (-1)

/* ---------------------------------------------------------------- binomials (Eq 5.6) */
/* C(v, k) by Pascal's rule, exact in uint64 (the caller keeps n small). */
static uint64_t **binom_table(int64_t n, int kmax) {
  uint64_t **c = (uint64_t **)malloc(sizeof(uint64_t *) * (size_t)(n + 1));
  for (int64_t v = 0; v <= n; v++) {
    c[v] = (uint64_t *)calloc((size_t)kmax + 1, sizeof(uint64_t));
    c[v][0] = 1;
    for (int k = 1; k <= kmax; k++) c[v][k] = v == 0 ? 0 : c[v - 1][k - 1] + c[v - 1][k];
  }
  return c;
}
static void binom_free(uint64_t **c, int64_t n) {
  for (int64_t v = 0; v <= n; v++) free(c[v]);
  free(c);
}

/* distance d(i, j) from the lower-distance vector: (i, j), i > j at i(i-1)/2 + j */
static float dist_lt(const float *lt, int64_t i, int64_t j) {
  if (i == j) return 0.0f;
  if (i < j) { int64_t t = i; i = j; j = t; }
  return lt[i * (i - 1) / 2 + j];
}

/* ---------------------------------------------------------------- simplices */
typedef struct {
  float diam;
  int dim;
  uint64_t cidx;
  int v[OR_MAXV]; /* vertices, strictly DEcreasing: v[0] > v[1] > ... (Remark 5.1.7) */
} simplex;

typedef struct {
  simplex *a;
  int64_t len, cap;
} simplex_vec;

static void sv_push(simplex_vec *s, const simplex *x) {
  if (s->len == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 1024;
    s->a = (simplex *)realloc(s->a, sizeof(simplex) * (size_t)s->cap);
  }
  s->a[s->len++] = *x;
}

/* Eq 5.6: cidx(v_d > ... > v_0) = sum_i C(v_i, i+1).  v[] holds v_d first. */
static uint64_t cidx_of(uint64_t **C, const int *v, int dim) {
  uint64_t c = 0;
  for (int p = 0; p <= dim; p++) c += C[v[p]][dim - p + 1];
  return c;
}

/* Enumerate every vertex subset of size k (dimension k-1) with diam <= t by plain
 * recursion over increasing vertex ids (chosen[0] < chosen[1] < ...).  The running
 * diameter is the max pairwise distance of the chosen prefix (Eq 5.3); a prefix over the
 * threshold cannot be extended (every superset has a larger-or-equal diameter). */
typedef struct {
  const float *lt;
  uint64_t **C;
  float thr;
  int k;
  int chosen[OR_MAXV];
  simplex_vec *out;
  int64_t n;
} enum_ctx;

static void enum_rec(enum_ctx *e, int depth, int64_t start, float diam) {
  if (depth == e->k) {
    simplex s;
    memset(&s, 0, sizeof s);
    s.dim = e->k - 1;
    s.diam = diam;
    for (int p = 0; p < e->k; p++) s.v[p] = e->chosen[e->k - 1 - p]; /* decreasing */
    s.cidx = cidx_of(e->C, s.v, s.dim);
    sv_push(e->out, &s);
    return;
  }
  for (int64_t v = start; v < e->n; v++) {
    float dm = diam;
    for (int p = 0; p < depth; p++) {
      float d = dist_lt(e->lt, v, e->chosen[p]);
      if (d > dm) dm = d;
    }
    if (!(dm <= e->thr)) continue; /* diam(s) <= t, inclusive (Eq 5.3; reading A7) */
    e->chosen[depth] = (int)v;
    enum_rec(e, depth + 1, v + 1, dm);
  }
}

/* §5.1.4 simplex-wise refinement: diam asc, then dim asc, then cidx DEscending. */
static int filtration_cmp(const void *pa, const void *pb) {
  const simplex *a = (const simplex *)pa, *b = (const simplex *)pb;
  if (a->diam < b->diam) return -1;
  if (a->diam > b->diam) return 1;
  if (a->dim != b->dim) return a->dim < b->dim ? -1 : 1;
  if (a->cidx != b->cidx) return a->cidx > b->cidx ? -1 : 1;
  return 0;
}

/* ---------------------------------------------------------------- Z/2 columns */
typedef struct {
  int32_t *r; /* sorted ascending row indices */
  int32_t len, cap;
} column;

static int col_low(const column *c) { return c->len ? c->r[c->len - 1] : NONE; } /* Eq 3.89 / A17 */

/* R[j] <- R[j] + R[i] over Z/2: symmetric difference of two sorted lists. */
static void col_add(column *dst, const column *src, int32_t **scratch, int32_t *scap) {
  int32_t need = dst->len + src->len;
  if (need > *scap) {
    *scap = need * 2;
    *scratch = (int32_t *)realloc(*scratch, sizeof(int32_t) * (size_t)*scap);
  }
  int32_t *o = *scratch;
  int32_t a = 0, b = 0, m = 0;
  while (a < dst->len && b < src->len) {
    if (dst->r[a] < src->r[b]) o[m++] = dst->r[a++];
    else if (dst->r[a] > src->r[b]) o[m++] = src->r[b++];
    else { a++; b++; } /* 1 + 1 = 0 */
  }
  while (a < dst->len) o[m++] = dst->r[a++];
  while (b < src->len) o[m++] = src->r[b++];
  if (m > dst->cap) {
    dst->cap = m;
    dst->r = (int32_t *)realloc(dst->r, sizeof(int32_t) * (size_t)m);
  }
  memcpy(dst->r, o, sizeof(int32_t) * (size_t)m);
  dst->len = m;
}

/* Alg 2, verbatim order of operations.  L[row] = owning column or NONE. */
static void standard_reduce(column *R, int64_t N, int32_t *L) {
  int32_t *scratch = NULL, scap = 0;
  for (int64_t i = 0; i < N; i++) L[i] = NONE;
  for (int64_t j = 0; j < N; j++) {
    while (R[j].len != 0 && L[col_low(&R[j])] != NONE) col_add(&R[j], &R[L[col_low(&R[j])]], &scratch, &scap);
    if (R[j].len != 0) L[col_low(&R[j])] = (int32_t)j;
  }
  free(scratch);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* ---------------------------------------------------------------- result handle */
typedef struct {
  int64_t len;
  float *birth, *death;
  uint64_t *bcidx, *dcidx; /* dcidx = UINT64_MAX for an essential class */
} pair_list;

typedef struct oracle_result {
  int max_dim;
  pair_list *pairs;     /* [max_dim+1] */
  int64_t *n_simplices; /* [max_dim+2]: #p-simplices with diam <= t */
} oracle_result;

static void pl_push(pair_list *p, int64_t *cap, float b, float d, uint64_t bc, uint64_t dc) {
  if (p->len == *cap) {
    *cap = *cap ? 2 * *cap : 64;
    p->birth = (float *)realloc(p->birth, sizeof(float) * (size_t)*cap);
    p->death = (float *)realloc(p->death, sizeof(float) * (size_t)*cap);
    p->bcidx = (uint64_t *)realloc(p->bcidx, sizeof(uint64_t) * (size_t)*cap);
    p->dcidx = (uint64_t *)realloc(p->dcidx, sizeof(uint64_t) * (size_t)*cap);
  }
  p->birth[p->len] = b;
  p->death[p->len] = d;
  p->bcidx[p->len] = bc;
  p->dcidx[p->len] = dc;
  p->len++;
}

/* Steps 1+2: every simplex of dim 0..top with diam <= t, sorted in §5.1.4 order. */
static simplex_vec build_filtration(const float *lt, int64_t n, int top, float thr, uint64_t **C) {
  simplex_vec all = {0};
  for (int k = 1; k <= top + 1; k++) {
    enum_ctx e;
    memset(&e, 0, sizeof e);
    e.lt = lt; e.C = C; e.thr = thr; e.k = k; e.out = &all; e.n = n;
    enum_rec(&e, 0, 0, 0.0f);
  }
  qsort(all.a, (size_t)all.len, sizeof(simplex), filtration_cmp);
  return all;
}

/* position lookup: per dimension, an array over cidx in [0, C(n, dim+1)) */
static int32_t **build_position_index(const simplex_vec *all, int64_t n, int top, uint64_t **C) {
  int32_t **pos = (int32_t **)calloc((size_t)top + 1, sizeof(int32_t *));
  for (int k = 0; k <= top; k++) {
    uint64_t m = (uint64_t)(k + 1) <= (uint64_t)n ? C[n][k + 1] : 0;
    pos[k] = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    for (uint64_t i = 0; i < m; i++) pos[k][i] = NONE;
  }
  for (int64_t j = 0; j < all->len; j++) pos[all->a[j].dim][all->a[j].cidx] = (int32_t)j;
  return pos;
}

/* Step 3: column j = positions of the facets of simplex j (Def 2.6.7). */
static column *build_boundary(const simplex_vec *all, int32_t **pos, uint64_t **C) {
  column *R = (column *)calloc((size_t)all->len, sizeof(column));
  for (int64_t j = 0; j < all->len; j++) {
    const simplex *s = &all->a[j];
    if (s->dim == 0) continue;
    R[j].cap = R[j].len = s->dim + 1;
    R[j].r = (int32_t *)malloc(sizeof(int32_t) * (size_t)R[j].cap);
    for (int drop = 0; drop <= s->dim; drop++) {
      int f[OR_MAXV], m = 0;
      for (int p = 0; p <= s->dim; p++)
        if (p != drop) f[m++] = s->v[p];
      int32_t fp = pos[s->dim - 1][cidx_of(C, f, s->dim - 1)];
      if (fp == NONE) { fprintf(stderr, "oracle: facet missing (not a complex)\n"); abort(); }
      R[j].r[drop] = fp;
    }
    qsort(R[j].r, (size_t)R[j].len, sizeof(int32_t), cmp_i32);
  }
  return R;
}

/* error codes mirror the product's meaning but are the oracle's own */
#define OR_OK 0
#define OR_EINVAL 1
#define OR_ECAP 3

oracle_result *oracle_barcode(const float *lt, int64_t n, int max_dim, float threshold, int *err) {
  *err = OR_OK;
  if (n < 1 || max_dim < 0 || max_dim + 2 > OR_MAXV || !lt || threshold != threshold || threshold < 0) {
    *err = OR_EINVAL;
    return NULL;
  }
  int top = max_dim + 1; /* the (D+1)-skeleton: dim-(D+1) simplices kill dim-D classes */
  uint64_t **C = binom_table(n, top + 1);
  for (int k = 0; k <= top; k++)
    if ((int64_t)k + 1 <= n && C[n][k + 1] > (uint64_t)200000000) { /* oracle is for small inputs */
      binom_free(C, n);
      *err = OR_ECAP;
      return NULL;
    }
  simplex_vec all = build_filtration(lt, n, top, threshold, C);
  int32_t **pos = build_position_index(&all, n, top, C);
  column *R = build_boundary(&all, pos, C);
  int32_t *L = (int32_t *)malloc(sizeof(int32_t) * (size_t)(all.len ? all.len : 1));
  standard_reduce(R, all.len, L);

  oracle_result *res = (oracle_result *)calloc(1, sizeof(oracle_result));
  res->max_dim = max_dim;
  res->pairs = (pair_list *)calloc((size_t)max_dim + 1, sizeof(pair_list));
  res->n_simplices = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
  int64_t *caps = (int64_t *)calloc((size_t)max_dim + 1, sizeof(int64_t));
  for (int64_t j = 0; j < all.len; j++) res->n_simplices[all.a[j].dim]++;
  /* Step 5a: pivots -> finite pairs [diam(low(j)), diam(j)) in dim(low(j)) */
  for (int64_t j = 0; j < all.len; j++) {
    int lo = col_low(&R[j]);
    if (lo == NONE) continue;
    const simplex *b = &all.a[lo], *d = &all.a[j];
    if (b->dim <= max_dim) pl_push(&res->pairs[b->dim], &caps[b->dim], b->diam, d->diam, b->cidx, d->cidx);
  }
  /* Step 5b: neither a pivot row nor a nonzero column -> essential [diam(i), +inf) */
  for (int64_t i = 0; i < all.len; i++) {
    const simplex *b = &all.a[i];
    if (b->dim > max_dim) continue;
    if (R[i].len == 0 && L[i] == NONE) pl_push(&res->pairs[b->dim], &caps[b->dim], b->diam, INFINITY, b->cidx, UINT64_MAX);
  }
  free(caps);
  for (int64_t j = 0; j < all.len; j++) free(R[j].r);
  free(R);
  free(L);
  for (int k = 0; k <= top; k++) free(pos[k]);
  free(pos);
  free(all.a);
  binom_free(C, n);
  return res;
}

int oracle_max_dim(const oracle_result *r) { return r->max_dim; }
int64_t oracle_num_pairs(const oracle_result *r, int dim) { return (dim < 0 || dim > r->max_dim) ? 0 : r->pairs[dim].len; }
int64_t oracle_num_simplices(const oracle_result *r, int dim) { return (dim < 0 || dim > r->max_dim + 1) ? 0 : r->n_simplices[dim]; }
void oracle_get_pairs(const oracle_result *r, int dim, float *birth, float *death, uint64_t *bcidx, uint64_t *dcidx) {
  const pair_list *p = &r->pairs[dim];
  memcpy(birth, p->birth, sizeof(float) * (size_t)p->len);
  memcpy(death, p->death, sizeof(float) * (size_t)p->len);
  memcpy(bcidx, p->bcidx, sizeof(uint64_t) * (size_t)p->len);
  memcpy(dcidx, p->dcidx, sizeof(uint64_t) * (size_t)p->len);
}
void oracle_free(oracle_result *r) {
  if (!r) return;
  for (int d = 0; d <= r->max_dim; d++) {
    free(r->pairs[d].birth); free(r->pairs[d].death); free(r->pairs[d].bcidx); free(r->pairs[d].dcidx);
  }
  free(r->pairs);
  free(r->n_simplices);
  free(r);
}

/* ---------------------------------------------------------------- Def 5.3.4 */
static int cidx_cmp(const void *pa, const void *pb) {
  uint64_t a = ((const simplex *)pa)->cidx, b = ((const simplex *)pb)->cidx;
  return (a > b) - (a < b);
}

/* For every d-simplex s with diam <= t (in cidx order): apparent flag and partner cidx.
 * t_old = the OLDEST cofacet of s in the complex (the first in §5.1.4 order: smallest
 * diameter, ties -> LARGEST cidx); s is apparent iff s is the YOUNGEST facet of t_old
 * (the last in §5.1.4 order: largest diameter, ties -> SMALLEST cidx).
 * Returns the number of d-simplices written (call with out == NULL to size). */
int64_t oracle_apparent(const float *lt, int64_t n, int d, float threshold, uint64_t *out_cidx, int8_t *out_flag,
                        uint64_t *out_partner) {
  if (n < 1 || d < 0 || d + 2 > OR_MAXV) return -1;
  uint64_t **C = binom_table(n, d + 2);
  simplex_vec sv = {0};
  enum_ctx e;
  memset(&e, 0, sizeof e);
  e.lt = lt; e.C = C; e.thr = threshold; e.k = d + 1; e.out = &sv; e.n = n;
  enum_rec(&e, 0, 0, 0.0f);
  int64_t m = sv.len;
  if (out_cidx) {
    qsort(sv.a, (size_t)m, sizeof(simplex), cidx_cmp); /* canonical output order: cidx ascending */
    for (int64_t i = 0; i < m; i++) {
      const simplex *s = &sv.a[i];
      /* all cofacets s + {v} in the complex */
      int have = 0;
      simplex best;
      memset(&best, 0, sizeof best);
      for (int64_t v = 0; v < n; v++) {
        int inside = 0;
        for (int p = 0; p <= d; p++) inside |= (s->v[p] == v);
        if (inside) continue;
        simplex t;
        memset(&t, 0, sizeof t);
        t.dim = d + 1;
        int q = 0, placed = 0;
        for (int p = 0; p <= d; p++) {
          if (!placed && v > s->v[p]) { t.v[q++] = (int)v; placed = 1; }
          t.v[q++] = s->v[p];
        }
        if (!placed) t.v[q++] = (int)v;
        float dm = 0.0f;
        for (int a = 0; a <= d + 1; a++)
          for (int b = a + 1; b <= d + 1; b++) {
            float x = dist_lt(lt, t.v[a], t.v[b]);
            if (x > dm) dm = x;
          }
        if (!(dm <= threshold)) continue;
        t.diam = dm;
        t.cidx = cidx_of(C, t.v, d + 1);
        if (!have || filtration_cmp(&t, &best) < 0) { best = t; have = 1; } /* oldest */
      }
      int8_t flag = 0;
      uint64_t partner = UINT64_MAX;
      if (have) {
        simplex young;
        memset(&young, 0, sizeof young);
        int hy = 0;
        for (int drop = 0; drop <= d + 1; drop++) {
          simplex f;
          memset(&f, 0, sizeof f);
          f.dim = d;
          int q = 0;
          for (int p = 0; p <= d + 1; p++)
            if (p != drop) f.v[q++] = best.v[p];
          float dm = 0.0f;
          for (int a = 0; a <= d; a++)
            for (int b = a + 1; b <= d; b++) {
              float x = dist_lt(lt, f.v[a], f.v[b]);
              if (x > dm) dm = x;
            }
          f.diam = dm;
          f.cidx = cidx_of(C, f.v, d);
          if (!hy || filtration_cmp(&f, &young) > 0) { young = f; hy = 1; } /* youngest */
        }
        if (young.cidx == s->cidx) { flag = 1; partner = best.cidx; }
      }
      out_cidx[i] = s->cidx;
      out_flag[i] = flag;
      out_partner[i] = partner;
    }
  }
  free(sv.a);
  binom_free(C, n);
  return m;
}

/* Def 5.3.4 for ONE d-simplex given by its vertices (any order), by brute force over its
 * explicit cofacets and their facets — usable at full problem sizes on sampled simplices.
 * Returns 1 and the partner's cidx if (s, t) is apparent, 0 if not, -1 if s is not in the
 * complex (diam > t). */
int oracle_apparent_one(const float *lt, int64_t n, int d, float threshold, const int *verts, uint64_t *partner) {
  if (d < 0 || d + 2 > OR_MAXV) return -1;
  uint64_t **C = binom_table(n, d + 2);
  simplex s;
  memset(&s, 0, sizeof s);
  s.dim = d;
  for (int p = 0; p <= d; ++p) s.v[p] = verts[p];
  for (int a = 0; a <= d; ++a) /* sort decreasing */
    for (int b = a + 1; b <= d; ++b)
      if (s.v[b] > s.v[a]) { int t = s.v[a]; s.v[a] = s.v[b]; s.v[b] = t; }
  float ds = 0.0f;
  for (int a = 0; a <= d; ++a)
    for (int b = a + 1; b <= d; ++b) { float x = dist_lt(lt, s.v[a], s.v[b]); if (x > ds) ds = x; }
  if (!(ds <= threshold)) { binom_free(C, n); return -1; }
  s.diam = ds;
  s.cidx = cidx_of(C, s.v, d);
  int have = 0;
  simplex best;
  memset(&best, 0, sizeof best);
  for (int64_t v = 0; v < n; v++) {
    int inside = 0;
    for (int p = 0; p <= d; ++p) inside |= (s.v[p] == v);
    if (inside) continue;
    simplex t;
    memset(&t, 0, sizeof t);
    t.dim = d + 1;
    int q = 0, placed = 0;
    for (int p = 0; p <= d; ++p) {
      if (!placed && v > s.v[p]) { t.v[q++] = (int)v; placed = 1; }
      t.v[q++] = s.v[p];
    }
    if (!placed) t.v[q++] = (int)v;
    float dm = 0.0f;
    for (int a = 0; a <= d + 1; a++)
      for (int b = a + 1; b <= d + 1; b++) { float x = dist_lt(lt, t.v[a], t.v[b]); if (x > dm) dm = x; }
    if (!(dm <= threshold)) continue;
    t.diam = dm;
    t.cidx = cidx_of(C, t.v, d + 1);
    if (!have || filtration_cmp(&t, &best) < 0) { best = t; have = 1; } /* oldest cofacet */
  }
  int res = 0;
  if (have) {
    simplex young;
    memset(&young, 0, sizeof young);
    int hy = 0;
    for (int drop = 0; drop <= d + 1; drop++) {
      simplex f;
      memset(&f, 0, sizeof f);
      f.dim = d;
      int q = 0;
      for (int p = 0; p <= d + 1; p++)
        if (p != drop) f.v[q++] = best.v[p];
      float dm = 0.0f;
      for (int a = 0; a <= d; a++)
        for (int b = a + 1; b <= d; b++) { float x = dist_lt(lt, f.v[a], f.v[b]); if (x > dm) dm = x; }
      f.diam = dm;
      f.cidx = cidx_of(C, f.v, d);
      if (!hy || filtration_cmp(&f, &young) > 0) { young = f; hy = 1; } /* youngest facet */
    }
    if (young.cidx == s.cidx) { res = 1; if (partner) *partner = best.cidx; }
  }
  binom_free(C, n);
  return res;
}

/* ---------------------------------------------------------------- Alg 2 alone */
/* Explicit matrix in CSC (col_ptr[ncols+1], rows[] ascending per column).  Writes the
 * final low of every column (NONE = -1 for a zero column).  Used for the Fig 4.1 pin. */
int oracle_reduce_columns(int64_t ncols, const int64_t *col_ptr, const int32_t *rows, int32_t *out_low) {
  column *R = (column *)calloc((size_t)(ncols ? ncols : 1), sizeof(column));
  for (int64_t j = 0; j < ncols; j++) {
    int64_t a = col_ptr[j], b = col_ptr[j + 1];
    R[j].len = R[j].cap = (int32_t)(b - a);
    R[j].r = (int32_t *)malloc(sizeof(int32_t) * (size_t)(R[j].cap ? R[j].cap : 1));
    for (int64_t k = a; k < b; k++) {
      if (rows[k] < 0 || rows[k] >= ncols) { for (int64_t q = 0; q <= j; q++) free(R[q].r); free(R); return OR_EINVAL; }
      R[j].r[k - a] = rows[k];
    }
    qsort(R[j].r, (size_t)R[j].len, sizeof(int32_t), cmp_i32);
  }
  int32_t *L = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ncols ? ncols : 1));
  standard_reduce(R, ncols, L);
  for (int64_t j = 0; j < ncols; j++) out_low[j] = col_low(&R[j]);
  for (int64_t j = 0; j < ncols; j++) free(R[j].r);
  free(R);
  free(L);
  return OR_OK;
}

/* ---------------------------------------------------------------- enclosing radius */
/* §5.2.12: R = min_x max_y d(x, y); n = 1 -> 0 (A27). */
float oracle_enclosing_radius(const float *lt, int64_t n) {
  if (n < 2) return 0.0f;
  float best = INFINITY;
  for (int64_t i = 0; i < n; i++) {
    float mx = 0.0f;
    for (int64_t j = 0; j < n; j++) {
      float x = dist_lt(lt, i, j);
      if (x > mx) mx = x;
    }
    if (mx < best) best = mx;
  }
  return best;
}
