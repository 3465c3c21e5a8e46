/*
 * hgr_oracle.c -- TEST INFRASTRUCTURE ONLY (see hgr_oracle.h).
 *
 * Plain-C restatement of the reference's CPU algorithm. Each function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/include/hgr/). Arithmetic order inside every loop
 * follows the reference so that results agree to the last few ulps (bitwise
 * when both are compiled without FMA contraction).
 */
#include "hgr_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

const char* hgro_last_error(void) { return g_err; }

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

/* ---- grid hierarchy (grid_hierarchy.hpp:33-188) --------------------------- */

static int is_pow2_plus_1(size_t n) { return n >= 2 && (((n - 1) & (n - 2)) == 0); }

static int ctz_size(size_t v) {
  int c = 0;
  while (!(v & 1u)) { v >>= 1; ++c; }
  return c;
}

static double coord(const hgro_grid* g, int d, size_t i) {
  return g->coords[d] ? g->coords[d][i] : (double)i;
}

/* GridHierarchy ctor validation (grid_hierarchy.hpp:51-70) */
int hgro_levels(const hgro_grid* g) {
  if (g->rank < 1 || g->rank > 3) return fail("grid must have 1 to 3 dimensions");
  int min_depth = -1;
  for (int d = 0; d < g->rank; ++d) {
    if (!is_pow2_plus_1(g->n[d])) {
      snprintf(g_err, sizeof g_err, "dimension size must be 2^k+1 (dimension %d has %zu nodes)",
               d, g->n[d]);
      return -1;
    }
    for (size_t i = 0; i + 1 < g->n[d]; ++i)
      if (!(coord(g, d, i) < coord(g, d, i + 1))) {
        snprintf(g_err, sizeof g_err,
                 "coordinates must be strictly increasing (dimension %d)", d);
        return -1;
      }
    int depth = ctz_size(g->n[d] - 1);
    if (min_depth < 0 || depth < min_depth) min_depth = depth;
  }
  return min_depth;
}

static size_t level_stride(int L, int l) { return (size_t)1 << (unsigned)(L - l); }

/* level_extent (grid_hierarchy.hpp:105-107), padded to rank 3 (ndarray.hpp:90-94) */
static void level_ext(const hgro_grid* g, int L, int l, size_t e[3]) {
  for (int d = 0; d < 3; ++d)
    e[d] = d < g->rank ? (g->n[d] - 1) / level_stride(L, l) + 1 : 1;
}

/* natural_strides (ndarray.hpp:80-88) of the finest array */
static void nat_strides(const hgro_grid* g, size_t s[3]) {
  size_t acc = 1;
  s[0] = s[1] = s[2] = 0;
  for (int d = g->rank - 1; d >= 0; --d) {
    s[d] = acc;
    acc *= g->n[d];
  }
}

/* spacings(level, d) (grid_hierarchy.hpp:163-177): h_i = x_{(i+1)s} - x_{is} */
static double* spacings(const hgro_grid* g, int L, int l, int d, size_t* count) {
  size_t s = level_stride(L, l);
  size_t n = (g->n[d] - 1) / s;
  double* h = (double*)malloc((n ? n : 1) * sizeof(double));
  for (size_t i = 0; i < n; ++i) h[i] = coord(g, d, (i + 1) * s) - coord(g, d, i * s);
  *count = n;
  return h;
}

typedef struct {
  double to_left, to_right;
} nweights;

/* refined_weights(level, d) (grid_hierarchy.hpp:178-187, :27-31), in double */
static nweights* refined_weights(const hgro_grid* g, int L, int l, int d) {
  size_t nh;
  double* h = spacings(g, L, l, d, &nh);
  nweights* w = (nweights*)malloc((nh / 2 + 1) * sizeof(nweights));
  for (size_t q = 0; q < nh / 2; ++q) {
    const double span = h[2 * q] + h[2 * q + 1];
    w[q].to_left = h[2 * q + 1] / span;
    w[q].to_right = h[2 * q] / span;
  }
  free(h);
  return w;
}

size_t hgro_class_node_count(const hgro_grid* g, int cls) {
  int L = hgro_levels(g);
  if (L < 0 || cls < 0 || cls > L) return 0;
  size_t e[3], c[3];
  level_ext(g, L, cls, e);
  size_t n = e[0] * e[1] * e[2];
  if (cls == 0) return n;
  level_ext(g, L, cls - 1, c);
  return n - c[0] * c[1] * c[2];
}

/* ---- precision-generic part ------------------------------------------------- */

enum { RF_SUB = 0, RF_ADD = 1, RF_SET = 2, RF_DIFF = 3 };

#define T double
#define SUF f64
#include "hgr_oracle_impl.inc"
#undef T
#undef SUF

#define T float
#define SUF f32
#include "hgr_oracle_impl.inc"
#undef T
#undef SUF
