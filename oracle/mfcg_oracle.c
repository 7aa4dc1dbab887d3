/*
 * mfcg_oracle.c -- CPU oracle, C restatement.  TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Restates, loop for loop, the reference's algorithm for the hot path
 * (/root/reference/pkg/src/mfcg; the reference itself is pure Python/NumPy and has no
 * compiled sources, so there is no oracle/_ref to build):
 *   cell kernel        operator.py:253-281  (evaluate_gradients tensor.py:335-347, flux einsum
 *                      operator.py:271-274, integrate_gradients tensor.py:357-370), plain S/D
 *                      matrices (tensor.py:291: identical to the even-odd form up to reassociation)
 *   apply              operator.py:338-360  (gather with constrained entries zeroed, scatter-add
 *                      dropping constrained rows, identity rows)
 *   merged (P)CG       solvers.py:601-792   in its three-phase sequentially-equivalent form
 *   fused reductions   solvers.py:112-127
 * Parity: pinned against oracle/mfcg_oracle.py and the reference fixtures in
 * tests/test_oracle.py::test_c_oracle_*.  POSIX threads over cells / vector entries (the image has
 * no libgomp); the scatter uses atomic adds, so results vary at the 1e-16 level between runs
 * with more than one thread.
 *
 * Used for: mid-size parity of the GPU path (sizes the NumPy oracle cannot finish in seconds) and
 * as the CPU baseline of bench.py (all host threads).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define MAXN 10

typedef struct {
  int p, nq;
  int64_t n_cells, n_dofs;
  const int64_t* idx;        /* [n_cells][(p+1)^3] expanded indices (dofs.py:215-218) */
  const unsigned char* cmask; /* [n_dofs] constrained flag */
  const double* S;           /* [nq][p+1] */
  const double* D;           /* [nq][p+1] */
  const double* G;           /* [per_cell ? n_cells : 1][nq^3][6] xx,yy,zz,xy,xz,yz (mesh.py:194-201) */
  int per_cell;
} oracle_problem;

static int g_threads = 0;
int oracle_max_threads(void) {
  if (g_threads > 0) return g_threads;
  const char* e = getenv("MFCG_ORACLE_THREADS");
  long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 256) n = 256;
  g_threads = (int)n;
  return g_threads;
}
void oracle_set_threads(int n) { g_threads = n > 0 ? n : 0; }

typedef void (*range_fn)(int64_t lo, int64_t hi, int tid, void* ctx);
typedef struct { range_fn fn; int64_t lo, hi; int tid; void* ctx; } task_t;
static void* task_main(void* a) { task_t* t = (task_t*)a; t->fn(t->lo, t->hi, t->tid, t->ctx); return NULL; }
/* static block partition of [0, n) over the worker threads */
static void parallel_for(int64_t n, range_fn fn, void* ctx) {
  int nt = oracle_max_threads();
  if (n < 4096 || nt == 1) { fn(0, n, 0, ctx); return; }
  pthread_t th[256];
  task_t tk[256];
  for (int t = 0; t < nt; ++t) {
    tk[t].fn = fn; tk[t].lo = n * t / nt; tk[t].hi = n * (t + 1) / nt; tk[t].tid = t; tk[t].ctx = ctx;
    if (t > 0) pthread_create(&th[t], NULL, task_main, &tk[t]);
  }
  task_main(&tk[0]);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}
static void atomic_add_double(double* addr, double val) {
  uint64_t* a = (uint64_t*)addr;
  uint64_t old = __atomic_load_n(a, __ATOMIC_RELAXED), neu;
  do {
    double d;
    memcpy(&d, &old, 8);
    d += val;
    memcpy(&neu, &d, 8);
  } while (!__atomic_compare_exchange_n(a, &old, neu, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED));
}

/* out[c][b][a'] = sum_a M[a'][a] in[c][b][a] along direction dir of an (nc x nb x na) -> tensor;
   generic 1D contraction over the chosen axis of a [n2][n1][n0] array (0 = x fastest). */
static void sweep(const double* M, int mo, int mi, int transpose, int dir, const int* dims_in,
                  const double* in, double* out) {
  int di[3] = {dims_in[0], dims_in[1], dims_in[2]};
  int dout[3] = {di[0], di[1], di[2]};
  dout[dir] = mo;
  for (int c = 0; c < dout[2]; ++c)
    for (int b = 0; b < dout[1]; ++b)
      for (int a = 0; a < dout[0]; ++a) {
        int o[3] = {a, b, c};
        double acc = 0.0;
        for (int t = 0; t < mi; ++t) {
          int s[3] = {a, b, c};
          s[dir] = t;
          const double m = transpose ? M[t * mo + o[dir]] : M[o[dir] * mi + t];
          acc += m * in[(s[2] * di[1] + s[1]) * di[0] + s[0]];
        }
        out[(c * dout[1] + b) * dout[0] + a] = acc;
      }
}

/* local = A_e u for one cell (operator.py:253-281) */
static void cell_laplacian(const oracle_problem* pb, const double* G, const double* u, double* local) {
  const int n = pb->p + 1, nq = pb->nq, nq3 = nq * nq * nq;
  double t1[MAXN * MAXN * MAXN], t2[MAXN * MAXN * MAXN];
  double grad[3][MAXN * MAXN * MAXN], flux[3][MAXN * MAXN * MAXN];
  for (int c = 0; c < 3; ++c) { /* evaluate_gradients: D in direction c, S elsewhere */
    int d0[3] = {n, n, n};
    sweep(c == 0 ? pb->D : pb->S, nq, n, 0, 0, d0, u, t1);
    int d1[3] = {nq, n, n};
    sweep(c == 1 ? pb->D : pb->S, nq, n, 0, 1, d1, t1, t2);
    int d2[3] = {nq, nq, n};
    sweep(c == 2 ? pb->D : pb->S, nq, n, 0, 2, d2, t2, grad[c]);
  }
  for (int q = 0; q < nq3; ++q) { /* flux = G grad, G symmetric 6-storage */
    const double* g = G + 6 * (int64_t)q;
    const double gx = grad[0][q], gy = grad[1][q], gz = grad[2][q];
    flux[0][q] = g[0] * gx + g[3] * gy + g[4] * gz;
    flux[1][q] = g[3] * gx + g[1] * gy + g[5] * gz;
    flux[2][q] = g[4] * gx + g[5] * gy + g[2] * gz;
  }
  const int n3 = n * n * n;
  for (int i = 0; i < n3; ++i) local[i] = 0.0;
  for (int c = 0; c < 3; ++c) { /* integrate_gradients: transposed sweeps, summed over c */
    int d0[3] = {nq, nq, nq};
    sweep(c == 0 ? pb->D : pb->S, n, nq, 1, 0, d0, flux[c], t1);
    int d1[3] = {n, nq, nq};
    sweep(c == 1 ? pb->D : pb->S, n, nq, 1, 1, d1, t1, t2);
    int d2[3] = {n, n, nq};
    sweep(c == 2 ? pb->D : pb->S, n, nq, 1, 2, d2, t2, t1);
    for (int i = 0; i < n3; ++i) local[i] += t1[i];
  }
}

typedef struct { const oracle_problem* pb; const double* src; double* dst; } apply_ctx;
static void apply_zero(int64_t lo, int64_t hi, int tid, void* c) {
  apply_ctx* a = (apply_ctx*)c; (void)tid;
  for (int64_t i = lo; i < hi; ++i) a->dst[i] = 0.0;
}
static void apply_cells(int64_t lo, int64_t hi, int tid, void* cc) {
  apply_ctx* a = (apply_ctx*)cc; (void)tid;
  const oracle_problem* pb = a->pb;
  const int n = pb->p + 1, n3 = n * n * n, nq3 = pb->nq * pb->nq * pb->nq;
  double u[MAXN * MAXN * MAXN], local[MAXN * MAXN * MAXN];
  for (int64_t c = lo; c < hi; ++c) {
    const int64_t* id = pb->idx + c * n3;
    for (int i = 0; i < n3; ++i) u[i] = pb->cmask[id[i]] ? 0.0 : a->src[id[i]];   /* operator.py:341-342 */
    cell_laplacian(pb, pb->G + (pb->per_cell ? c * 6 * (int64_t)nq3 : 0), u, local);
    for (int i = 0; i < n3; ++i)
      if (!pb->cmask[id[i]]) atomic_add_double(&a->dst[id[i]], local[i]);        /* operator.py:348-353 */
  }
}
static void apply_identity(int64_t lo, int64_t hi, int tid, void* c) {
  apply_ctx* a = (apply_ctx*)c; (void)tid;
  for (int64_t i = lo; i < hi; ++i)
    if (a->pb->cmask[i]) a->dst[i] = a->src[i];                                   /* operator.py:359-360 */
}
/* dst = A src (operator.py:294-360) */
void oracle_apply(const oracle_problem* pb, const double* src, double* dst) {
  apply_ctx a = {pb, src, dst};
  parallel_for(pb->n_dofs, apply_zero, &a);
  parallel_for(pb->n_cells, apply_cells, &a);
  parallel_for(pb->n_dofs, apply_identity, &a);
}

typedef struct {
  const double *b, *minv; double *x, *r, *p, *v;
  double am1, bm1, xc2, c2; int xmode, simple;
  double part[256][8];
} cg_ctx;
static void cg_init(int64_t lo, int64_t hi, int tid, void* cc) {
  cg_ctx* c = (cg_ctx*)cc; double bb = 0.0;
  for (int64_t i = lo; i < hi; ++i) { c->r[i] = c->b[i]; c->x[i] = 0.0; c->p[i] = 0.0; c->v[i] = 0.0; bb += c->b[i] * c->b[i]; }
  c->part[tid][0] = bb;
}
static void cg_pre(int64_t lo, int64_t hi, int tid, void* cc) {                    /* solvers.py:660-690 */
  cg_ctx* c = (cg_ctx*)cc; (void)tid;
  for (int64_t i = lo; i < hi; ++i) {
    if (c->xmode == 2) c->x[i] += c->am1 * c->p[i] + c->xc2 * (c->p[i] - c->minv[i] * c->r[i]);
    else if (c->xmode == 1) c->x[i] += c->am1 * c->p[i];
    c->r[i] -= c->am1 * c->v[i];
    c->p[i] = c->minv[i] * c->r[i] + c->bm1 * c->p[i];
  }
}
static void cg_post(int64_t lo, int64_t hi, int tid, void* cc) {                   /* solvers.py:112-127 */
  cg_ctx* c = (cg_ctx*)cc; double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = lo; i < hi; ++i) {
    const double r = c->r[i], p = c->p[i], v = c->v[i], mr = c->minv[i] * r, mv = c->minv[i] * v;
    s[0] += r * r; s[1] += p * v; s[2] += r * v; s[3] += v * v; s[4] += r * mr; s[5] += r * mv; s[6] += v * mv;
  }
  for (int q = 0; q < 7; ++q) c->part[tid][q] = s[q];
}
static void cg_final(int64_t lo, int64_t hi, int tid, void* cc) {                  /* solvers.py:771-782 */
  cg_ctx* c = (cg_ctx*)cc; (void)tid;
  for (int64_t i = lo; i < hi; ++i)
    c->x[i] += c->simple ? c->am1 * c->p[i] : c->am1 * c->p[i] + c->c2 * (c->p[i] - c->minv[i] * c->r[i]);
}

/* merged Jacobi-PCG, fixed iteration count, three-phase form (solvers.py:601-792).
   history: [iters][4] alpha, beta, gamma, residual.  Returns iterations done (negative: breakdown). */
int oracle_combined_pcg(const oracle_problem* pb, const double* b, const double* minv, int iters, double tol,
                        double* x, double* history) {
  const int64_t n = pb->n_dofs;
  const int nt = (n < 4096) ? 1 : oracle_max_threads();
  cg_ctx* c = (cg_ctx*)calloc(1, sizeof(cg_ctx));
  c->b = b; c->minv = minv; c->x = x;
  c->r = (double*)malloc(sizeof(double) * n);
  c->p = (double*)malloc(sizeof(double) * n);
  c->v = (double*)malloc(sizeof(double) * n);
  parallel_for(n, cg_init, c);
  double bb = 0.0;
  for (int t = 0; t < nt; ++t) bb += c->part[t][0];
  const double bnorm = sqrt(bb);
  double am1 = 0, bm1 = 0, am2 = 0, bm2 = 0, residual = 1.0;
  int stagnant = 0, k = 0, done = 0;
  if (bnorm > 0.0) {
    for (k = 1; k <= iters; ++k) {
      const int live = am1 != 0.0 || am2 != 0.0;
      c->xmode = (k > 1 && live && (k & 1)) ? ((am2 != 0.0 && bm2 != 0.0) ? 2 : 1) : 0;
      c->xc2 = c->xmode == 2 ? am2 / bm2 : 0.0;
      c->am1 = am1; c->bm1 = bm1;
      parallel_for(n, cg_pre, c);
      oracle_apply(pb, c->p, c->v);
      memset(c->part, 0, sizeof(c->part));
      parallel_for(n, cg_post, c);
      double s[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int t = 0; t < nt; ++t) for (int q = 0; q < 7; ++q) s[q] += c->part[t][q];
      double alpha = 0.0, beta = 0.0;
      if (stagnant) residual = sqrt(s[0]) / bnorm;
      else if (s[0] == 0.0) { residual = 0.0; stagnant = 1; }
      else if (s[4] <= 0.0) { done = -k; break; }
      else if (s[1] <= 0.0) { if (residual < tol) stagnant = 1; else { done = -k; break; } }
      else {
        alpha = s[4] / s[1];
        beta = (s[4] - 2.0 * alpha * s[5] + alpha * alpha * s[6]) / s[4];
        const double stop_sq = s[0] - 2.0 * alpha * s[2] + alpha * alpha * s[3];
        residual = sqrt(stop_sq > 0.0 ? stop_sq : 0.0) / bnorm;
        if (beta <= 0.0) { if (residual < tol) stagnant = 1; else { done = -k; break; } }
      }
      if (history) { double* h = history + 4 * (int64_t)(k - 1); h[0] = alpha; h[1] = beta; h[2] = s[0]; h[3] = residual; }
      am2 = am1; bm2 = bm1; am1 = alpha; bm1 = beta;
      done = k;
    }
    if (done > 0) {
      c->simple = (done & 1) || am2 == 0.0 || bm2 == 0.0;
      c->c2 = c->simple ? 0.0 : am2 / bm2;
      c->am1 = am1;
      parallel_for(n, cg_final, c);
    }
  }
  free(c->r); free(c->p); free(c->v); free(c);
  return done;
}
