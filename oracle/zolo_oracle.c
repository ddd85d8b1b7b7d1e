/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Zolotarev filter path.
 *
 * A plain-C11 restatement of the reference's hot path (ZoloEig,
 * /root/reference/proj/include/zoloeig), used only by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg, always as the
 * checker and never as the measured or shipped path. The product
 * (paper_1701_08935_b200/) never links or loads this file.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function below
 * against golden vectors emitted by the unmodified reference
 * (oracle/_ref/libzoloref.so, built by oracle/Makefile; fixtures in
 * tests/golden/, generator tests/golden/make_golden.py). The loops keep the
 * reference's operation order, so with the same compiler flags (-O3, no FMA
 * contraction) most results agree bit for bit.
 *
 * Layout conventions follow the reference: dense blocks are column-major,
 * complex values interleaved (re, im) exactly like std::complex<double>
 * (dense.hpp:53-115); CSR uses int64 offsets/indices (sparse.hpp:31-36).
 *
 * Restated functions (reference file:line):
 *   or_spmv              sparse.hpp:113-129
 *   or_assemble_shifted  sparse.hpp:153-186
 *   or_rcm               rcm.hpp:33-115 (bfs_far_node + reorder_rcm)
 *   or_factorize         band_factor.hpp:135-182
 *   or_solve             band_factor.hpp:53-85
 *   or_adjoint_solve     band_factor.hpp:88-117
 *   or_op_create         filter_engine.hpp:40-45 + band_factor.hpp:199-220
 *   or_apply_g           filter_engine.hpp:56-82
 *   hessenberg_ls        gmres.hpp:58-88
 *   multishift_column    gmres.hpp:98-182 (one column)
 *   or_apply_filter      filter_engine.hpp:86-155
 * Status codes: 0 ok, 1 domain, 2 numerical, 3 factorization, 4 gmres.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* ------------------------------------------------------------------ */
/* packed design offsets (shared with include/zolo_b200.h)              */
/* ------------------------------------------------------------------ */
enum {
  D_MHAT = 10,
  D_CONST = 13,
  D_OUTER_M = 17,
  D_HEAD = 19
};
static const double* d_inner_poles(const double* d, int r) { (void)r; return d + D_HEAD; }
static const double* d_inner_weights(const double* d, int r) { return d + D_HEAD + 2 * r; }
static const double* d_outer_pf(const double* d, int r) { return d + D_HEAD + 5 * r; }
static const double* d_outer_c(const double* d, int r) { return d + D_HEAD + 6 * r + (2 * r - 1); }

/* ------------------------------------------------------------------ */
/* CSR                                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t* rp;
  int64_t* ci;
  cplx* vc;   /* complex values, or NULL */
  double* vr; /* real values, or NULL */
} csr_t;

static void csr_free(csr_t* m) {
  free(m->rp);
  free(m->ci);
  free(m->vc);
  free(m->vr);
  memset(m, 0, sizeof(*m));
}

static csr_t csr_copy(int cx, int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  csr_t m;
  memset(&m, 0, sizeof(m));
  m.n = n;
  const int64_t nnz = rp[n];
  m.rp = malloc(sizeof(int64_t) * (n + 1));
  m.ci = malloc(sizeof(int64_t) * (nnz > 0 ? nnz : 1));
  memcpy(m.rp, rp, sizeof(int64_t) * (n + 1));
  memcpy(m.ci, ci, sizeof(int64_t) * nnz);
  if (cx) {
    m.vc = malloc(sizeof(cplx) * (nnz > 0 ? nnz : 1));
    for (int64_t k = 0; k < nnz; ++k) m.vc[k] = CMPLX(v[2 * k], v[2 * k + 1]);
  } else {
    m.vr = malloc(sizeof(double) * (nnz > 0 ? nnz : 1));
    memcpy(m.vr, v, sizeof(double) * nnz);
  }
  return m;
}

static csr_t csr_identity(int cx, int64_t n) {
  csr_t m;
  memset(&m, 0, sizeof(m));
  m.n = n;
  m.rp = malloc(sizeof(int64_t) * (n + 1));
  m.ci = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  if (cx) m.vc = malloc(sizeof(cplx) * (n > 0 ? n : 1));
  else m.vr = malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    m.rp[i] = i;
    m.ci[i] = i;
    if (cx) m.vc[i] = CMPLX(1.0, 0.0);
    else m.vr[i] = 1.0;
  }
  m.rp[n] = n;
  return m;
}

/* y = M x for a dense block; sparse.hpp:113-129. Complex in/out when either
 * side is complex (promote_t); x_cx/y_cx select the element type. */
static void spmv_block(const csr_t* m, int64_t k, const void* x, int x_cx, void* y) {
  const int out_cx = x_cx || (m->vc != NULL);
  const int64_t n = m->n;
  for (int64_t c = 0; c < k; ++c) {
    for (int64_t i = 0; i < n; ++i) {
      if (out_cx) {
        cplx s = 0;
        for (int64_t q = m->rp[i]; q < m->rp[i + 1]; ++q) {
          const cplx a = m->vc ? m->vc[q] : CMPLX(m->vr[q], 0.0);
          const int64_t j = m->ci[q] + c * n;
          const cplx b = x_cx ? ((const cplx*)x)[j] : CMPLX(((const double*)x)[j], 0.0);
          s += a * b;
        }
        ((cplx*)y)[i + c * n] = s;
      } else {
        double s = 0;
        for (int64_t q = m->rp[i]; q < m->rp[i + 1]; ++q)
          s += m->vr[q] * ((const double*)x)[m->ci[q] + c * n];
        ((double*)y)[i + c * n] = s;
      }
    }
  }
}

int or_spmv(int cx_mat, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
            int cx_x, int64_t k, const double* x, double* y) {
  csr_t m = csr_copy(cx_mat, n, rp, ci, v);
  spmv_block(&m, k, x, cx_x, y);
  csr_free(&m);
  return 0;
}

/* A - sigma B on the union pattern; sparse.hpp:153-186. b may be NULL (= I). */
static csr_t assemble_shifted(const csr_t* a, const csr_t* b, cplx sigma) {
  const int64_t n = a->n;
  csr_t out;
  memset(&out, 0, sizeof(out));
  out.n = n;
  const int64_t cap = a->rp[n] + b->rp[n] + 1;
  out.rp = calloc(n + 1, sizeof(int64_t));
  out.ci = malloc(sizeof(int64_t) * cap);
  out.vc = malloc(sizeof(cplx) * cap);
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t ka = a->rp[i], kb = b->rp[i];
    const int64_t ea = a->rp[i + 1], eb = b->rp[i + 1];
    while (ka < ea || kb < eb) {
      const int64_t ja = ka < ea ? a->ci[ka] : n;
      const int64_t jb = kb < eb ? b->ci[kb] : n;
      const cplx av = ka < ea ? (a->vc ? a->vc[ka] : CMPLX(a->vr[ka], 0.0)) : 0;
      const cplx bv = kb < eb ? (b->vc ? b->vc[kb] : CMPLX(b->vr[kb], 0.0)) : 0;
      if (ja < jb) {
        out.ci[nnz] = ja;
        out.vc[nnz++] = av;
        ++ka;
      } else if (jb < ja) {
        out.ci[nnz] = jb;
        out.vc[nnz++] = -sigma * bv;
        ++kb;
      } else {
        out.ci[nnz] = ja;
        out.vc[nnz++] = av - sigma * bv;
        ++ka;
        ++kb;
      }
    }
    out.rp[i + 1] = nnz;
  }
  return out;
}

/* ------------------------------------------------------------------ */
/* RCM; rcm.hpp:33-115                                                 */
/* ------------------------------------------------------------------ */
static const int64_t* g_sort_deg_rp;
static int cmp_deg_idx(const void* x, const void* y) {
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  const int64_t da = g_sort_deg_rp[a + 1] - g_sort_deg_rp[a];
  const int64_t db = g_sort_deg_rp[b + 1] - g_sort_deg_rp[b];
  if (da != db) return da < db ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

static int64_t bfs_far_node(int64_t n, const int64_t* rp, const int64_t* ci, int64_t root,
                            int64_t* level, int64_t* queue) {
  for (int64_t i = 0; i < n; ++i) level[i] = -1;
  int64_t head = 0, tail = 0;
  queue[tail++] = root;
  level[root] = 0;
  int64_t far = root, far_level = 0;
  while (head < tail) {
    const int64_t u = queue[head++];
    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
      const int64_t v = ci[k];
      if (v != u && level[v] < 0) {
        level[v] = level[u] + 1;
        queue[tail++] = v;
        if (level[v] > far_level) {
          far_level = level[v];
          far = v;
        } else if (level[v] == far_level) {
          const int64_t du = rp[far + 1] - rp[far];
          const int64_t dv = rp[v + 1] - rp[v];
          if (dv < du || (dv == du && v < far)) far = v;
        }
      }
    }
  }
  return far;
}

int or_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm) {
  int64_t* level = malloc(sizeof(int64_t) * (n + 1));
  int64_t* queue = malloc(sizeof(int64_t) * (n + 1));
  int64_t* nbrs = malloc(sizeof(int64_t) * (n + 1));
  char* visited = calloc(n + 1, 1);
  int64_t count = 0;
  while (count < n) {
    int64_t root = n, best = INT64_MAX;
    for (int64_t v = 0; v < n; ++v)
      if (!visited[v] && rp[v + 1] - rp[v] < best) {
        best = rp[v + 1] - rp[v];
        root = v;
      }
    for (int it = 0; it < 2; ++it) root = bfs_far_node(n, rp, ci, root, level, queue);
    int64_t head = 0, tail = 0;
    queue[tail++] = root;
    visited[root] = 1;
    while (head < tail) {
      const int64_t u = queue[head++];
      perm[count++] = u;
      int64_t nn = 0;
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        const int64_t v = ci[k];
        if (v != u && !visited[v]) {
          visited[v] = 1;
          nbrs[nn++] = v;
        }
      }
      g_sort_deg_rp = rp;
      qsort(nbrs, nn, sizeof(int64_t), cmp_deg_idx);
      for (int64_t q = 0; q < nn; ++q) queue[tail++] = nbrs[q];
    }
  }
  for (int64_t i = 0; i < n / 2; ++i) {
    const int64_t t = perm[i];
    perm[i] = perm[n - 1 - i];
    perm[n - 1 - i] = t;
  }
  free(level);
  free(queue);
  free(nbrs);
  free(visited);
  return 0;
}

/* ------------------------------------------------------------------ */
/* banded LU; band_factor.hpp:135-182                                  */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n, bw;
  int64_t* ordering; /* new -> old */
  cplx* band;        /* band[j*(2bw+1) + bw + i - j] */
  double min_ratio;
} or_factor;

static int64_t bandwidth_under(const csr_t* m, const int64_t* pos) {
  int64_t bw = 0;
  for (int64_t i = 0; i < m->n; ++i)
    for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k) {
      const int64_t pi = pos[i], pj = pos[m->ci[k]];
      const int64_t d = pi > pj ? pi - pj : pj - pi;
      if (d > bw) bw = d;
    }
  return bw;
}

/* Returns NULL and sets *pivot_index on a rejected pivot. */
static or_factor* factorize(const csr_t* m, const int64_t* ordering, int64_t* pivot_index) {
  const int64_t n = m->n;
  int64_t* pos = malloc(sizeof(int64_t) * (n + 1));
  for (int64_t k = 0; k < n; ++k) pos[ordering[k]] = k;
  const int64_t bw = bandwidth_under(m, pos);
  const int64_t w = 2 * bw + 1;
  or_factor* f = calloc(1, sizeof(or_factor));
  f->n = n;
  f->bw = bw;
  f->ordering = malloc(sizeof(int64_t) * (n + 1));
  memcpy(f->ordering, ordering, sizeof(int64_t) * n);
  f->band = calloc((size_t)(w * n + 1), sizeof(cplx));
  double* row_norm = calloc(n + 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k) {
      const int64_t pi = pos[i], pj = pos[m->ci[k]];
      f->band[pj * w + bw + pi - pj] = m->vc[k];
      const double av = cabs(m->vc[k]);
      if (av > row_norm[pi]) row_norm[pi] = av;
    }
  double min_ratio = INFINITY;
  for (int64_t k = 0; k < n; ++k) {
    const cplx piv = f->band[k * w + bw];
    const double ratio = cabs(piv) / fmax(row_norm[k], 1e-300);
    if (ratio < min_ratio) min_ratio = ratio;
    if (!(cabs(piv) > 1e-14 * row_norm[k])) {
      if (pivot_index) *pivot_index = k;
      free(pos);
      free(row_norm);
      free(f->ordering);
      free(f->band);
      free(f);
      return NULL;
    }
    const int64_t hi = (n - 1 < k + bw) ? n - 1 : k + bw;
    cplx* colk = f->band + k * w + bw - k;
    const cplx inv = 1.0 / piv;
    for (int64_t i = k + 1; i <= hi; ++i) colk[i] *= inv;
    for (int64_t j = k + 1; j <= hi; ++j) {
      const cplx ukj = f->band[j * w + bw + k - j];
      if (ukj == 0) continue;
      cplx* colj = f->band + j * w + bw - j;
      for (int64_t i = k + 1; i <= hi; ++i) colj[i] -= colk[i] * ukj;
    }
  }
  f->min_ratio = min_ratio;
  free(pos);
  free(row_norm);
  return f;
}

static void factor_free(or_factor* f) {
  if (!f) return;
  free(f->ordering);
  free(f->band);
  free(f);
}

/* band_factor.hpp:53-85; rhs/out n x k complex, x is n scratch */
static void factor_solve(const or_factor* f, int64_t k, const cplx* rhs, cplx* out, cplx* x) {
  const int64_t n = f->n, bw = f->bw, w = 2 * bw + 1;
  for (int64_t c = 0; c < k; ++c) {
    const cplx* b = rhs + c * n;
    for (int64_t i = 0; i < n; ++i) x[i] = b[f->ordering[i]];
    for (int64_t j = 0; j < n; ++j) {
      const cplx xj = x[j];
      if (xj != 0) {
        const int64_t hi = (n - 1 < j + bw) ? n - 1 : j + bw;
        const cplx* col = f->band + j * w + bw - j;
        for (int64_t i = j + 1; i <= hi; ++i) x[i] -= col[i] * xj;
      }
    }
    for (int64_t j = n; j-- > 0;) {
      const int64_t w0 = j * w + bw - j;
      x[j] /= f->band[w0 + j];
      const cplx xj = x[j];
      if (xj != 0) {
        const int64_t lo = j > bw ? j - bw : 0;
        const cplx* col = f->band + w0;
        for (int64_t i = lo; i < j; ++i) x[i] -= col[i] * xj;
      }
    }
    cplx* o = out + c * n;
    for (int64_t i = 0; i < n; ++i) o[f->ordering[i]] = x[i];
  }
}

/* band_factor.hpp:88-117 */
static void factor_adjoint_solve(const or_factor* f, int64_t k, const cplx* rhs, cplx* out,
                                 cplx* x) {
  const int64_t n = f->n, bw = f->bw, w = 2 * bw + 1;
  for (int64_t c = 0; c < k; ++c) {
    const cplx* b = rhs + c * n;
    for (int64_t i = 0; i < n; ++i) x[i] = b[f->ordering[i]];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t lo = i > bw ? i - bw : 0;
      const cplx* coli = f->band + i * w + bw - i;
      cplx s = x[i];
      for (int64_t j = lo; j < i; ++j) s -= conj(coli[j]) * x[j];
      x[i] = s / conj(coli[i]);
    }
    for (int64_t i = n; i-- > 0;) {
      const int64_t hi = (n - 1 < i + bw) ? n - 1 : i + bw;
      const cplx* coli = f->band + i * w + bw - i;
      cplx s = x[i];
      for (int64_t j = i + 1; j <= hi; ++j) s -= conj(coli[j]) * x[j];
      x[i] = s;
    }
    cplx* o = out + c * n;
    for (int64_t i = 0; i < n; ++i) o[f->ordering[i]] = x[i];
  }
}

/* ------------------------------------------------------------------ */
/* filter operator                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
  int cx, r;
  int64_t n;
  csr_t a, b;
  int b_identity;
  or_factor** factors;
  int64_t* ordering;
  cplx* eff_w;
  double constant_term, outer_m;
  double* outer_pf;
  double* outer_root; /* sqrt(outer.c[2j]) */
  int64_t inner_solves, g_apps;
} or_op;

/* Factorization at one shift with the RCM ordering of the pattern of A - iB
 * (band_factor.hpp:199-220). */
static int build_factor(const csr_t* a, const csr_t* b, cplx sigma, const int64_t* ordering,
                        or_factor** out, int64_t* pivot_index) {
  csr_t s = assemble_shifted(a, b, sigma);
  *out = factorize(&s, ordering, pivot_index);
  csr_free(&s);
  return *out ? 0 : 3;
}

static int64_t* shared_ordering(const csr_t* a, const csr_t* b) {
  csr_t probe = assemble_shifted(a, b, CMPLX(0.0, 1.0));
  int64_t* ord = malloc(sizeof(int64_t) * (a->n + 1));
  or_rcm(a->n, probe.rp, probe.ci, ord);
  csr_free(&probe);
  return ord;
}

void or_op_free(or_op* op) {
  if (!op) return;
  for (int j = 0; j < op->r; ++j) factor_free(op->factors ? op->factors[j] : NULL);
  free(op->factors);
  free(op->ordering);
  free(op->eff_w);
  free(op->outer_pf);
  free(op->outer_root);
  csr_free(&op->a);
  csr_free(&op->b);
  free(op);
}

or_op* or_op_create(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                    const int64_t* brp, const int64_t* bci, const double* bv,
                    const double* design, int r, int* status, int64_t* pivot_index) {
  or_op* op = calloc(1, sizeof(or_op));
  op->cx = cx;
  op->r = r;
  op->n = n;
  op->a = csr_copy(cx, n, arp, aci, av);
  op->b_identity = brp == NULL;
  op->b = brp ? csr_copy(cx, n, brp, bci, bv) : csr_identity(cx, n);
  op->ordering = shared_ordering(&op->a, &op->b);
  op->factors = calloc(r, sizeof(or_factor*));
  const double* poles = d_inner_poles(design, r);
  const double* wts = d_inner_weights(design, r);
  op->eff_w = malloc(sizeof(cplx) * r);
  op->outer_pf = malloc(sizeof(double) * r);
  op->outer_root = malloc(sizeof(double) * r);
  const double m_hat = design[D_MHAT];
  for (int j = 0; j < r; ++j) {
    if (build_factor(&op->a, &op->b, CMPLX(poles[2 * j], poles[2 * j + 1]), op->ordering,
                     &op->factors[j], pivot_index) != 0) {
      *status = 3;
      or_op_free(op);
      return NULL;
    }
    op->eff_w[j] = m_hat * CMPLX(wts[2 * j], wts[2 * j + 1]);
    op->outer_pf[j] = d_outer_pf(design, r)[j];
    op->outer_root[j] = sqrt(d_outer_c(design, r)[2 * j]);
  }
  op->constant_term = design[D_CONST];
  op->outer_m = design[D_OUTER_M];
  *status = 0;
  return op;
}

void or_counters(const or_op* op, int64_t* out) {
  out[0] = op->inner_solves;
  out[1] = op->g_apps;
}

/* filter_engine.hpp:56-82 on an n x k block (S = double or complex). */
static void apply_g_block(or_op* op, int64_t k, const void* v, void* out) {
  const int64_t n = op->n, len = n * k;
  const int r = op->r;
  op->g_apps += 1;
  cplx* bvx = malloc(sizeof(cplx) * (len + 1));
  cplx* x = malloc(sizeof(cplx) * (len + 1));
  cplx* xa = malloc(sizeof(cplx) * (len + 1));
  cplx* scratch = malloc(sizeof(cplx) * (n + 1));
  if (op->cx) {
    const cplx* vv = v;
    cplx* acc = out;
    for (int64_t q = 0; q < len; ++q) acc[q] = op->constant_term * vv[q];
    if (op->b_identity)
      memcpy(bvx, vv, sizeof(cplx) * len);
    else
      spmv_block(&op->b, k, vv, 1, bvx);
    for (int j = 0; j < r; ++j) {
      factor_solve(op->factors[j], k, bvx, x, scratch);
      factor_adjoint_solve(op->factors[j], k, bvx, xa, scratch);
      const cplx w = op->eff_w[j];
      for (int64_t q = 0; q < len; ++q) acc[q] += w * x[q] + conj(w) * xa[q];
    }
    op->inner_solves += 2 * r;
  } else {
    const double* vv = v;
    double* acc = out;
    for (int64_t q = 0; q < len; ++q) acc[q] = op->constant_term * vv[q];
    if (op->b_identity) {
      for (int64_t q = 0; q < len; ++q) bvx[q] = CMPLX(vv[q], 0.0);
    } else {
      double* tmp = malloc(sizeof(double) * (len + 1));
      spmv_block(&op->b, k, vv, 0, tmp);
      for (int64_t q = 0; q < len; ++q) bvx[q] = CMPLX(tmp[q], 0.0);
      free(tmp);
    }
    for (int j = 0; j < r; ++j) {
      factor_solve(op->factors[j], k, bvx, x, scratch);
      const cplx w = op->eff_w[j];
      for (int64_t q = 0; q < len; ++q) acc[q] += 2.0 * creal(w * x[q]);
    }
    op->inner_solves += r;
  }
  free(bvx);
  free(x);
  free(xa);
  free(scratch);
}

int or_apply_g(or_op* op, int64_t k, const double* v, double* out) {
  apply_g_block(op, k, v, out);
  return 0;
}

/* gmres.hpp:58-88: min ||(H_m + s I) y - beta e1|| by Givens from scratch.
 * h is (ldh x *) column-major, real (hr) or complex (hc). Returns |g_m|. */
static double hessenberg_ls(const double* hr, const cplx* hc, int64_t ldh, int64_t m, cplx s,
                            double beta, cplx* y, cplx* t, cplx* g) {
  const int64_t ldt = m + 1;
  for (int64_t j = 0; j < m; ++j) {
    for (int64_t i = 0; i <= m; ++i) t[i + j * ldt] = 0;
    const int64_t top = j + 1 < m ? j + 1 : m;
    for (int64_t i = 0; i <= top; ++i)
      t[i + j * ldt] = hc ? hc[i + j * ldh] : CMPLX(hr[i + j * ldh], 0.0);
  }
  for (int64_t j = 0; j < m; ++j) t[j + j * ldt] += s;
  for (int64_t i = 0; i <= m; ++i) g[i] = 0;
  g[0] = beta;
  for (int64_t j = 0; j < m; ++j) {
    const cplx a = t[j + j * ldt], b = t[j + 1 + j * ldt];
    const double na = creal(a) * creal(a) + cimag(a) * cimag(a);
    const double nb = creal(b) * creal(b) + cimag(b) * cimag(b);
    const double nr = sqrt(na + nb);
    if (nr == 0.0) continue;
    const cplx c = a / nr, sn = b / nr;
    for (int64_t k = j; k < m; ++k) {
      const cplx t0 = t[j + k * ldt], t1 = t[j + 1 + k * ldt];
      t[j + k * ldt] = conj(c) * t0 + conj(sn) * t1;
      t[j + 1 + k * ldt] = -sn * t0 + c * t1;
    }
    const cplx g0 = g[j], g1 = g[j + 1];
    g[j] = conj(c) * g0 + conj(sn) * g1;
    g[j + 1] = -sn * g0 + c * g1;
  }
  for (int64_t i = m; i-- > 0;) {
    cplx v = g[i];
    for (int64_t k = i + 1; k < m; ++k) v -= t[i + k * ldt] * y[k];
    y[i] = v / t[i + i * ldt];
  }
  return cabs(g[m]);
}

/* One column of multishift_gmres (gmres.hpp:98-182) with the filter's shift
 * set; writes the combined filter output column (filter_engine.hpp:109-126).
 * Returns m; res/conv per shift. */
static int64_t filter_column(or_op* op, double tol, int64_t max_iter, const void* rhs, void* out,
                             double* res_out, int* conv_out, int64_t* op_apps) {
  const int64_t n = op->n;
  const int cx = op->cx;
  const int r = op->r, q = 2 * r;
  cplx* shifts = malloc(sizeof(cplx) * q);
  for (int j = 0; j < r; ++j) {
    shifts[2 * j] = CMPLX(0.0, op->outer_root[j]);
    shifts[2 * j + 1] = CMPLX(0.0, -op->outer_root[j]);
  }
  const size_t es = cx ? sizeof(cplx) : sizeof(double);
  double beta = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (cx) {
      const cplx z = ((const cplx*)rhs)[t];
      beta += creal(z) * creal(z) + cimag(z) * cimag(z);
    } else {
      const double z = ((const double*)rhs)[t];
      beta += z * z;
    }
  }
  beta = sqrt(beta);
  cplx** sols = calloc(q, sizeof(cplx*));
  for (int k = 0; k < q; ++k) sols[k] = calloc(n + 1, sizeof(cplx));
  int64_t m = 0;
  int happy = 0;
  double* shift_res = calloc(q, sizeof(double));
  int* shift_done = calloc(q, sizeof(int));
  cplx** shift_y = calloc(q, sizeof(cplx*));
  int64_t* shift_len = calloc(q, sizeof(int64_t));
  char** basis = NULL;
  int64_t nbasis = 0;
  double* hr = NULL;
  cplx* hc = NULL;
  const int64_t ldh = max_iter + 1;
  if (beta != 0.0) {
    basis = calloc(max_iter + 2, sizeof(char*));
    basis[0] = malloc(es * (n + 1));
    for (int64_t t = 0; t < n; ++t) {
      if (cx) ((cplx*)basis[0])[t] = CMPLX(1.0 / beta, 0.0) * ((const cplx*)rhs)[t];
      else ((double*)basis[0])[t] = (1.0 / beta) * ((const double*)rhs)[t];
    }
    nbasis = 1;
    if (cx) hc = calloc(ldh * max_iter + 1, sizeof(cplx));
    else hr = calloc(ldh * max_iter + 1, sizeof(double));
    char* w = malloc(es * (n + 1));
    cplx* ytmp = malloc(sizeof(cplx) * (max_iter + 1));
    cplx* tws = malloc(sizeof(cplx) * (max_iter + 2) * (max_iter + 1));
    cplx* gws = malloc(sizeof(cplx) * (max_iter + 2));
    while (m < max_iter) {
      apply_g_block(op, 1, basis[m], w);
      ++*op_apps;
      for (int pass = 0; pass < 2; ++pass) {
        for (int64_t i = 0; i <= m; ++i) {
          if (cx) {
            const cplx* vi = (const cplx*)basis[i];
            cplx* wc = (cplx*)w;
            cplx hij = 0;
            for (int64_t t = 0; t < n; ++t) hij += conj(vi[t]) * wc[t];
            for (int64_t t = 0; t < n; ++t) wc[t] -= hij * vi[t];
            hc[i + m * ldh] += hij;
          } else {
            const double* vi = (const double*)basis[i];
            double* wc = (double*)w;
            double hij = 0;
            for (int64_t t = 0; t < n; ++t) hij += vi[t] * wc[t];
            for (int64_t t = 0; t < n; ++t) wc[t] -= hij * vi[t];
            hr[i + m * ldh] += hij;
          }
        }
      }
      double wn = 0;
      for (int64_t t = 0; t < n; ++t) {
        if (cx) {
          const cplx z = ((cplx*)w)[t];
          wn += creal(z) * creal(z) + cimag(z) * cimag(z);
        } else {
          const double z = ((double*)w)[t];
          wn += z * z;
        }
      }
      wn = sqrt(wn);
      if (cx) hc[m + 1 + m * ldh] = CMPLX(wn, 0.0);
      else hr[m + 1 + m * ldh] = wn;
      ++m;
      if (wn > 1e-14 * beta) {
        basis[nbasis] = malloc(es * (n + 1));
        for (int64_t t = 0; t < n; ++t) {
          if (cx) ((cplx*)basis[nbasis])[t] = CMPLX(1.0 / wn, 0.0) * ((cplx*)w)[t];
          else ((double*)basis[nbasis])[t] = (1.0 / wn) * ((double*)w)[t];
        }
        ++nbasis;
      } else {
        happy = 1;
      }
      int all_done = 1;
      for (int k = 0; k < q; ++k) {
        if (shift_done[k]) continue;
        const double rs = hessenberg_ls(hr, hc, ldh, m, shifts[k], beta, ytmp, tws, gws);
        free(shift_y[k]);
        shift_y[k] = malloc(sizeof(cplx) * (m + 1));
        memcpy(shift_y[k], ytmp, sizeof(cplx) * m);
        shift_len[k] = m;
        shift_res[k] = rs / beta;
        if (shift_res[k] <= tol) shift_done[k] = 1;
        all_done = all_done && shift_done[k];
      }
      if (all_done || happy) break;
    }
    free(w);
    free(ytmp);
    free(tws);
    free(gws);
    for (int k = 0; k < q; ++k) {
      cplx* xc = sols[k];
      for (int64_t i = 0; i < m && i < shift_len[k]; ++i) {
        const cplx yi = shift_y[k][i];
        for (int64_t t = 0; t < n; ++t) {
          const cplx vt = cx ? ((const cplx*)basis[i])[t] : CMPLX(((const double*)basis[i])[t], 0.0);
          xc[t] += yi * vt;
        }
      }
    }
  }
  for (int k = 0; k < q; ++k) {
    res_out[k] = shift_res[k];
    conv_out[k] = (shift_res[k] <= tol) || happy || beta == 0.0;
  }
  /* filter_engine.hpp:112-126 */
  for (int64_t t = 0; t < n; ++t) {
    cplx yv = 0;
    for (int j = 0; j < r; ++j) {
      const double aj = op->outer_pf[j];
      yv += 0.5 * aj * (sols[2 * j][t] + sols[2 * j + 1][t]);
    }
    const double vt_r = cx ? 0 : ((const double*)rhs)[t];
    const cplx vt = cx ? ((const cplx*)rhs)[t] : CMPLX(vt_r, 0.0);
    const cplx val = 0.5 * op->outer_m * yv + 0.5 * vt;
    if (cx) ((cplx*)out)[t] = val;
    else ((double*)out)[t] = creal(val);
  }
  for (int64_t i = 0; i < nbasis; ++i) free(basis[i]);
  free(basis);
  free(hr);
  free(hc);
  for (int k = 0; k < q; ++k) {
    free(sols[k]);
    free(shift_y[k]);
  }
  free(sols);
  free(shift_y);
  free(shift_len);
  free(shift_res);
  free(shift_done);
  free(shifts);
  return m;
}

/* filter_engine.hpp:86-155 (serial column order). Report merge as :127-133.
 * Returns 4 when any shift failed to converge (GmresError). */
int or_apply_filter(or_op* op, double tol, int64_t max_iter, int64_t k, const double* v,
                    double* y, int64_t* col_iters, double* residuals, int32_t* converged,
                    int64_t* iters, int64_t* op_apps) {
  const int64_t n = op->n;
  const int q = 2 * op->r;
  const size_t es = op->cx ? 2 : 1;
  double* res = malloc(sizeof(double) * q);
  int* conv = malloc(sizeof(int) * q);
  for (int s = 0; s < q; ++s) {
    residuals[s] = 0.0;
    converged[s] = 1;
  }
  *iters = 0;
  *op_apps = 0;
  int status = 0;
  for (int64_t c = 0; c < k; ++c) {
    const int64_t m =
        filter_column(op, tol, max_iter, v + c * n * es, y + c * n * es, res, conv, op_apps);
    col_iters[c] = m;
    if (m > *iters) *iters = m;
    for (int s = 0; s < q; ++s) {
      if (res[s] > residuals[s]) residuals[s] = res[s];
      if (!conv[s]) {
        converged[s] = 0;
        status = 4;
      }
    }
  }
  free(res);
  free(conv);
  return status;
}

/* Convenience: factor (A - sigma B) with the shared RCM ordering and run
 * solve/adjoint_solve on an n x k complex rhs; mirrors zr_shifted_solve. */
int or_shifted_solve(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                     const int64_t* brp, const int64_t* bci, const double* bv, double sig_re,
                     double sig_im, int64_t k, const double* rhs, double* x, double* xa,
                     int64_t* perm_out, int64_t* bw_out, double* min_ratio,
                     int64_t* pivot_index) {
  csr_t a = csr_copy(cx, n, arp, aci, av);
  csr_t b = brp ? csr_copy(cx, n, brp, bci, bv) : csr_identity(cx, n);
  int64_t* ord = shared_ordering(&a, &b);
  if (perm_out) memcpy(perm_out, ord, sizeof(int64_t) * n);
  or_factor* f = NULL;
  if (pivot_index) *pivot_index = -1;
  const int st = build_factor(&a, &b, CMPLX(sig_re, sig_im), ord, &f, pivot_index);
  if (st == 0) {
    if (bw_out) *bw_out = f->bw;
    if (min_ratio) *min_ratio = f->min_ratio;
    cplx* scratch = malloc(sizeof(cplx) * (n + 1));
    if (x) factor_solve(f, k, (const cplx*)rhs, (cplx*)x, scratch);
    if (xa) factor_adjoint_solve(f, k, (const cplx*)rhs, (cplx*)xa, scratch);
    free(scratch);
  }
  factor_free(f);
  free(ord);
  csr_free(&a);
  csr_free(&b);
  return st;
}
