// mfcg_b200.cu -- C ABI (include/mfcg_b200.h) and the degree-independent host
// logic: context, brick numbering, permutation between the caller's numbering
// and the brick numbering, constraint mask.
#include <algorithm>
#include <new>

#include "mfcg_engine.cuh"

namespace mfcg {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }

EngineBase* make_engine_p1(OpCommon*, int*);
EngineBase* make_engine_p2(OpCommon*, int*);
EngineBase* make_engine_p3(OpCommon*, int*);
EngineBase* make_engine_p4(OpCommon*, int*);
EngineBase* make_engine_p5(OpCommon*, int*);
EngineBase* make_engine_p6(OpCommon*, int*);
EngineBase* make_engine_p7(OpCommon*, int*);
EngineBase* make_engine_p8(OpCommon*, int*);

EngineBase* make_engine(OpCommon* c, int* status) {
  switch (c->p) {
    case 1: return make_engine_p1(c, status);
    case 2: return make_engine_p2(c, status);
    case 3: return make_engine_p3(c, status);
    case 4: return make_engine_p4(c, status);
    case 5: return make_engine_p5(c, status);
    case 6: return make_engine_p6(c, status);
    case 7: return make_engine_p7(c, status);
    case 8: return make_engine_p8(c, status);
  }
  set_error("degree must be in 1..8");
  *status = MFCG_EINVAL;
  return nullptr;
}

// default brick extent in x / y per geometry class and degree == Cfg<P, G>::BX / BY (mfcg_kernels.cuh)
static const int kBrickX[2][9] = {{0, 16, 10, 6, 5, 4, 3, 2, 2}, {0, 16, 10, 6, 5, 4, 3, 2, 2}};
static const int kBrickY[2][9] = {{0, 16, 10, 6, 5, 4, 3, 2, 2}, {0, 16, 10, 6, 5, 3, 2, 2, 2}};

}  // namespace mfcg

using namespace mfcg;

struct mfcg_ctx {
  Ctx c;
};

struct mfcg_op {
  OpCommon common;
  EngineBase* engine = nullptr;
};

extern "C" {

const char* mfcg_last_error(void) { return g_error.c_str(); }

int mfcg_ctx_create(int device, mfcg_ctx** out) {
  if (!out) { set_error("ctx out pointer is NULL"); return MFCG_EINVAL; }
  *out = nullptr;
  int count = 0;
  cudaError_t err = cudaGetDeviceCount(&count);
  if (err != cudaSuccess || count == 0) {
    set_error(std::string("no CUDA device available: ") + cudaGetErrorString(err));
    return MFCG_ECUDA;
  }
  if (device < 0 || device >= count) { set_error("device index out of range"); return MFCG_EINVAL; }
  MFCG_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  MFCG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    set_error("this library is built for sm_100a (B200) only");
    return MFCG_EUNSUPPORTED;
  }
  mfcg_ctx* ctx = new (std::nothrow) mfcg_ctx();
  if (!ctx) { set_error("out of host memory"); return MFCG_ENOMEM; }
  ctx->c.device = device;
  ctx->c.sm_count = prop.multiProcessorCount;
  MFCG_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
  *out = ctx;
  return MFCG_OK;
}

void* mfcg_ctx_stream(mfcg_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

void mfcg_ctx_destroy(mfcg_ctx* ctx) {
  if (!ctx) return;
  if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  delete ctx;
}

void mfcg_op_destroy(mfcg_op* op) {
  if (!op) return;
  cudaSetDevice(op->common.ctx->device);
  delete op->engine;
  OpCommon& c = op->common;
  if (c.d_perm) cudaFree(c.d_perm);
  if (c.d_ent_start) cudaFree(c.d_ent_start);
  if (c.d_mask) cudaFree(c.d_mask);
  if (c.d_io) cudaFree(c.d_io);
  if (c.d_invdiag) cudaFree(c.d_invdiag);
  if (c.d_state) cudaFree(c.d_state);
  if (c.h_state) cudaFreeHost(c.h_state);
  if (c.d_flag) cudaFree(c.d_flag);
  delete op;
}

static int op_create_impl(mfcg_ctx* ctx, const mfcg_op_desc* d, mfcg_op* op) {
  OpCommon& c = op->common;
  c.ctx = &ctx->c;
  const int p = d->degree, nq = d->n_q_1d;
  if (p < 1 || p > 8) { set_error("degree must be in 1..8"); return MFCG_EINVAL; }
  if (nq < p + 1) { set_error("n_q_1d must be at least p+1"); return MFCG_EINVAL; }
  if (nq != p + 1 && d->geometry == MFCG_GEOM_AFFINE) {
    // the separable path only needs M and K, any n_q works
  }
  if (nq > 10) { set_error("n_q_1d > 10 is not supported"); return MFCG_EUNSUPPORTED; }
  for (int k = 0; k < 3; ++k)
    if (d->cells[k] < 1 || !(d->extents[k] > 0)) { set_error("cells and extents must be positive"); return MFCG_EINVAL; }
  if (!d->shape_values || !d->shape_gradients || !d->quad_weights || !d->quad_points || !d->gl_weights ||
      !d->gl_gradients || !d->gl_points || !d->cell_index_blocks) {
    set_error("operator tables must not be NULL");
    return MFCG_EINVAL;
  }
  if (d->geometry == MFCG_GEOM_AFFINE && d->deformation != 0.0) {
    set_error("affine geometry requires an undeformed mesh");  // mesh.py:214-216
    return MFCG_EINVAL;
  }
  if (d->geometry < 0 || d->geometry > 3) { set_error("unknown geometry variant"); return MFCG_EINVAL; }
  if (d->precision != 0 && d->precision != 1) { set_error("precision must be 0 (fp64) or 1 (fp32)"); return MFCG_EINVAL; }
  const i64 NX = (i64)d->cells[0] * p + 1, NY = (i64)d->cells[1] * p + 1, NZ = (i64)d->cells[2] * p + 1;
  if (d->n_dofs != NX * NY * NZ) {
    set_error("vector length does not match handler");  // scalar problems only
    return MFCG_EINVAL;
  }
  if (d->n_dofs >= (i64)2147483647) { set_error("more than 2^31-1 DoFs per GPU are not supported"); return MFCG_EUNSUPPORTED; }
  c.p = p;
  c.nq = nq;
  c.precision = d->precision;
  c.geometry = d->geometry;
  c.deformation = d->deformation;
  c.n_cells = (i64)d->cells[0] * d->cells[1] * d->cells[2];
  c.S.assign(d->shape_values, d->shape_values + nq * (p + 1));
  c.D.assign(d->shape_gradients, d->shape_gradients + nq * (p + 1));
  c.xq.assign(d->quad_points, d->quad_points + nq);
  c.wq.assign(d->quad_weights, d->quad_weights + nq);
  c.glx.assign(d->gl_points, d->gl_points + (p + 1));
  c.glw.assign(d->gl_weights, d->gl_weights + (p + 1));
  c.glD.assign(d->gl_gradients, d->gl_gradients + (p + 1) * (p + 1));
  BrickGrid& g = c.grid;
  g.p = p;
  g.n_dofs = d->n_dofs;
  for (int k = 0; k < 3; ++k) {
    g.cells[k] = d->cells[k];
    c.extents[k] = d->extents[k];
    c.h[k] = d->extents[k] / d->cells[k];
  }
  // brick extents: x, y bounded by the kernel's shared-memory window; z free
  for (int k = 0; k < 2; ++k) {
    const int gclass = d->geometry == MFCG_GEOM_AFFINE ? 0 : 1;
    const int cap = k == 0 ? kBrickX[gclass][p] : kBrickY[gclass][p];
    int b = d->brick[k] > 0 ? d->brick[k] : cap;
    if (b > cap) { set_error("brick extent in x/y exceeds the kernel window for this degree"); return MFCG_EINVAL; }
    g.B[k] = std::min(b, g.cells[k]);
  }
  {
    int bz = d->brick[2] > 0 ? d->brick[2] : std::min(8, g.cells[2]);
    bz = std::min(bz, g.cells[2]);
    if (d->brick[2] <= 0) {
      auto count = [&](int z) {
        return (i64)((g.cells[0] + g.B[0] - 1) / g.B[0]) * ((g.cells[1] + g.B[1] - 1) / g.B[1]) *
               ((g.cells[2] + z - 1) / z);
      };
      while (bz > 1 && count(bz) < 4 * (i64)ctx->c.sm_count) bz = (bz + 1) / 2;
    }
    g.B[2] = bz;
  }
  for (int k = 0; k < 3; ++k) g.mb[k] = (g.cells[k] + g.B[k] - 1) / g.B[k];
  c.n_bricks = (i64)g.mb[0] * g.mb[1] * g.mb[2];

  // ---- brick numbering: all brick interiors first (brick order, x fastest), then every
  // shared macro entity in lexicographic (z, y, x) order of the macro lattice
  const int ex = 2 * g.mb[0] + 1, ey = 2 * g.mb[1] + 1, ez = 2 * g.mb[2] + 1;
  std::vector<int> len[3];
  for (int k = 0; k < 3; ++k) {
    len[k].resize(2 * g.mb[k] + 1);
    for (int s = 0; s <= 2 * g.mb[k]; ++s) {
      if (s % 2 == 0) len[k][s] = 1;
      else {
        const int m = s / 2;
        len[k][s] = p * std::min(g.B[k], g.cells[k] - m * g.B[k]) - 1;
      }
    }
  }
  std::vector<i64> start((size_t)ex * ey * ez);
  i64 acc = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int sz = 0; sz < ez; ++sz)
      for (int sy = 0; sy < ey; ++sy)
        for (int sx = 0; sx < ex; ++sx) {
          const bool interior = (sx & 1) && (sy & 1) && (sz & 1);
          if (interior != (pass == 0)) continue;
          start[((size_t)sz * ey + sy) * ex + sx] = acc;
          acc += (i64)len[0][sx] * len[1][sy] * len[2][sz];
        }
  {
    i64 ni = 0;
    for (int mz = 0; mz < g.mb[2]; ++mz)
      for (int my = 0; my < g.mb[1]; ++my)
        for (int mx = 0; mx < g.mb[0]; ++mx)
          ni += (i64)len[0][2 * mx + 1] * len[1][2 * my + 1] * len[2][2 * mz + 1];
    g.n_int = ni;
  }
  if (acc != g.n_dofs) { set_error("internal error: brick numbering does not cover the lattice"); return MFCG_ECUDA; }

  cudaStream_t st = ctx->c.stream;
  MFCG_CUDA(cudaMalloc(&c.d_ent_start, sizeof(i64) * start.size()));
  MFCG_CUDA(cudaMemcpyAsync(c.d_ent_start, start.data(), sizeof(i64) * start.size(), cudaMemcpyHostToDevice, st));
  g.ent_start = c.d_ent_start;
  const i64 n_sh = g.n_dofs - g.n_int;
  MFCG_CUDA(cudaMalloc(&c.d_mask, (size_t)std::max<i64>(n_sh, 1)));
  MFCG_CUDA(cudaMemsetAsync(c.d_mask, 0, (size_t)std::max<i64>(n_sh, 1), st));
  g.mask = c.d_mask;
  MFCG_CUDA(cudaMalloc(&c.d_perm, sizeof(int) * g.n_dofs));
  MFCG_CUDA(cudaMemsetAsync(c.d_perm, 0xff, sizeof(int) * g.n_dofs, st));
  MFCG_CUDA(cudaMalloc(&c.d_io, sizeof(double) * g.n_dofs));
  MFCG_CUDA(cudaMalloc(&c.d_state, sizeof(SolveState)));
  MFCG_CUDA(cudaMallocHost(&c.h_state, sizeof(SolveState)));
  MFCG_CUDA(cudaMalloc(&c.d_flag, sizeof(int)));
  MFCG_CUDA(cudaMemsetAsync(c.d_flag, 0, sizeof(int), st));

  const int vgrid = ctx->c.sm_count * 8;
  {
    int* d_blocks = nullptr;
    MFCG_CUDA(cudaMalloc(&d_blocks, sizeof(int) * 27 * c.n_cells));
    MFCG_CUDA(cudaMemcpyAsync(d_blocks, d->cell_index_blocks, sizeof(int) * 27 * c.n_cells, cudaMemcpyHostToDevice, st));
    k_build_perm<<<vgrid, 256, 0, st>>>(g, d_blocks, c.n_cells, c.d_perm);
    MFCG_CUDA(cudaGetLastError());
    MFCG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_blocks);
  }
  if (d->n_constrained > 0) {
    if (!d->constrained) { set_error("constrained list is NULL"); return MFCG_EINVAL; }
    i64* d_con = nullptr;
    MFCG_CUDA(cudaMalloc(&d_con, sizeof(i64) * d->n_constrained));
    MFCG_CUDA(cudaMemcpyAsync(d_con, d->constrained, sizeof(i64) * d->n_constrained, cudaMemcpyHostToDevice, st));
    k_mark_constrained<<<vgrid, 256, 0, st>>>(d->n_constrained, d_con, c.d_perm, g.n_int, c.d_mask, c.d_flag);
    MFCG_CUDA(cudaGetLastError());
    int flag = 0;
    MFCG_CUDA(cudaMemcpyAsync(&flag, c.d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFCG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_con);
    if (flag) {
      set_error("constrained DoFs must lie on the domain boundary (they do for every handler the reference builds)");
      return MFCG_EUNSUPPORTED;
    }
  }
  int est = MFCG_ECUDA;
  op->engine = make_engine(&c, &est);
  if (!op->engine) return est == MFCG_OK ? MFCG_ECUDA : est;
  MFCG_CUDA(cudaStreamSynchronize(st));
  return MFCG_OK;
}

int mfcg_op_create(mfcg_ctx* ctx, const mfcg_op_desc* desc, mfcg_op** out) {
  if (!ctx || !desc || !out) { set_error("NULL argument"); return MFCG_EINVAL; }
  *out = nullptr;
  cudaSetDevice(ctx->c.device);
  mfcg_op* op = new (std::nothrow) mfcg_op();
  if (!op) { set_error("out of host memory"); return MFCG_ENOMEM; }
  op->common.ctx = &ctx->c;
  int rc = op_create_impl(ctx, desc, op);
  if (rc != MFCG_OK) {
    mfcg_op_destroy(op);
    return rc;
  }
  *out = op;
  return MFCG_OK;
}

int mfcg_op_get_info(mfcg_op* op, mfcg_op_info* info) {
  if (!op || !info) { set_error("NULL argument"); return MFCG_EINVAL; }
  op->engine->info(info);
  return MFCG_OK;
}

int mfcg_op_device_permutation(mfcg_op* op, int32_t* perm_host) {
  if (!op || !perm_host) { set_error("NULL argument"); return MFCG_EINVAL; }
  cudaSetDevice(op->common.ctx->device);
  MFCG_CUDA(cudaMemcpy(perm_host, op->common.d_perm, sizeof(int) * op->common.grid.n_dofs, cudaMemcpyDeviceToHost));
  return MFCG_OK;
}

int mfcg_op_apply(mfcg_op* op, const double* src, double* dst, int location) {
  if (!op || !src || !dst) { set_error("NULL argument"); return MFCG_EINVAL; }
  cudaSetDevice(op->common.ctx->device);
  return op->engine->apply(src, dst, location);
}

int mfcg_op_diagonal(mfcg_op* op, double* inv_diag, int location) {
  if (!op || !inv_diag) { set_error("NULL argument"); return MFCG_EINVAL; }
  cudaSetDevice(op->common.ctx->device);
  return op->engine->diagonal(inv_diag, location);
}

int mfcg_op_geometry(mfcg_op* op, int kind, double* out_host, int64_t n_doubles) {
  if (!op || !out_host) { set_error("NULL argument"); return MFCG_EINVAL; }
  cudaSetDevice(op->common.ctx->device);
  return op->engine->geometry(kind, out_host, n_doubles);
}

int mfcg_solve(mfcg_op* op, const mfcg_solve_args* args, mfcg_solve_result* result) {
  if (!op || !args || !result) { set_error("NULL argument"); return MFCG_EINVAL; }
  cudaSetDevice(op->common.ctx->device);
  return op->engine->solve(args, result);
}

int mfcg_comm_unique_id(void* unique_id_128) {
  (void)unique_id_128;
  set_error("slab communication is not built yet in this round");
  return MFCG_EUNSUPPORTED;
}

int mfcg_ctx_init_comm(mfcg_ctx* ctx, const void* unique_id_128, int rank, int n_ranks) {
  (void)ctx; (void)unique_id_128; (void)rank; (void)n_ranks;
  set_error("slab communication is not built yet in this round");
  return MFCG_EUNSUPPORTED;
}

}  // extern "C"
