// mfcg_engine.cuh -- host-side engine: owns device memory, launches the kernels,
// runs the device-resident CG loops.  One Engine<P, T> per (degree, precision).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mfcg_b200.h"
#include "mfcg_kernels.cuh"
#include "mfcg_brick2.cuh"
#include "mfcg_cellpath.cuh"

namespace mfcg {

void set_error(const std::string& msg);

#define MFCG_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t err__ = (call);                                                             \
    if (err__ != cudaSuccess) {                                                             \
      set_error(std::string(#call) + ": " + cudaGetErrorString(err__));                     \
      return err__ == cudaErrorMemoryAllocation ? MFCG_ENOMEM : MFCG_ECUDA;                 \
    }                                                                                       \
  } while (0)

// Owners for objects created inside entry points that have early error returns.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  cudaError_t create() {
    cudaError_t e = cudaEventCreate(&a);
    return e != cudaSuccess ? e : cudaEventCreate(&b);
  }
};
template <typename T> struct DevBuf {
  T* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * (n ? n : 1)); }
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t comm_stream = nullptr;  // plane exchange, overlapped with interior bricks
  void* nccl_comm = nullptr;
  int rank = 0, n_ranks = 1;
};

// Everything mfcg_op_create derives that does not depend on the template arguments.
struct OpCommon {
  Ctx* ctx = nullptr;
  BrickGrid grid{};
  i64 n_cells = 0;
  int p = 1, nq = 2, precision = 0, geometry = 0;
  int ncomp = 1;  // vector components per node (1 or 3); grid.n_dofs counts nodes
  std::vector<double> S, D, xq, wq, glx, glw, glD;
  double extents[3] = {1, 1, 1}, h[3] = {1, 1, 1}, deformation = 0.0;
  i64 n_bricks = 0;
  int slab_z0 = 0, global_cells_z = 0;
  bool has_lower = false, has_upper = false;  // neighbouring slabs below / above
  int* d_perm = nullptr;
  i64* d_ent_start = nullptr;
  unsigned char* d_mask = nullptr;
  double* d_io = nullptr;       // fp64 staging in caller numbering
  double* d_invdiag = nullptr;  // cached 1/diag, brick numbering, fp64
  SolveState* d_state = nullptr;
  SolveState* h_state = nullptr;  // pinned
  int* d_flag = nullptr;
};

struct EngineBase {
  virtual ~EngineBase() {}
  virtual int apply(const double* src, double* dst, int location) = 0;
  virtual int diagonal(double* out, int location) = 0;
  virtual int solve(const mfcg_solve_args* a, mfcg_solve_result* r) = 0;
  virtual void info(mfcg_op_info* out) = 0;
  virtual int geometry(int kind, double* out_host, i64 n_doubles) = 0;
  // ---- slab-group driver interface (mfcg_solve_group, mfcg_b200.cu)
  virtual int g_alloc() = 0;
  virtual bool g_has_diag() = 0;
  virtual int g_diag_local() = 0;
  virtual int g_diag_finish() = 0;
  virtual int g_begin(const mfcg_solve_args* a, int limit) = 0;
  virtual int g_set_state(const mfcg_solve_args* a, int limit, const double* global_bb_dev) = 0;
  virtual int g_front(bool diag_planes) = 0;
  virtual int g_unpack(bool diag_planes) = 0;
  virtual int g_post() = 0;
  virtual int g_scalar(const double* global_sums_dev) = 0;
  virtual int g_poll(int* active) = 0;
  virtual int g_end(const mfcg_solve_args* a, mfcg_solve_result* r) = 0;
  virtual void* g_plane(int side, int recv) = 0;
  virtual size_t g_plane_bytes(bool diag_planes) = 0;
  virtual double* g_sums() = 0;
  virtual int g_apply_front(const double* src, int location) = 0;
  virtual int g_apply_end(double* dst, int location) = 0;
  // standard (P)CG on slabs: the regions of solvers.py:296-336, dot products over owned DoFs
  virtual int g_std_begin(const mfcg_solve_args* a, int limit) = 0;
  virtual int g_std_init_vectors() = 0;
  virtual int g_std_init_scalar(const double* global_sums_dev) = 0;
  virtual int g_std_apply_front() = 0;
  virtual int g_std_apply_end() = 0;
  virtual int g_std_dot_pv() = 0;
  virtual int g_std_alpha_update(const double* global_sums_dev) = 0;
  virtual int g_std_dots_r() = 0;
  virtual int g_std_beta_p(const double* global_sums_dev) = 0;
};

template <int P, typename T>
class Engine : public EngineBase {
 public:
  static constexpr int N = P + 1;
  static constexpr int VT = 256;  // threads of the vector kernels

  explicit Engine(OpCommon* c) : c_(c) {}

  ~Engine() override {
    for (T** v : {&x_, &r_, &p_, &v_, &z_, &minv_}) if (*v) cudaFree(*v);
    if (partials_a_) cudaFree(partials_a_);
    if (partials_b_) cudaFree(partials_b_);
    if (d_history_) cudaFree(d_history_);
    if (geo_a_) cudaFree(geo_a_);
    if (geo_b_) cudaFree(geo_b_);
    for (void** b : {&plane_[0][0], &plane_[0][1], &plane_[1][0], &plane_[1][1]}) if (*b) cudaFree(*b);
    if (d_sums_) cudaFree(d_sums_);
    if (diag_raw_) cudaFree(diag_raw_);
    if (ev_front_) cudaEventDestroy(ev_front_);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
  }

  int init() {
    const double det = c_->h[0] * c_->h[1] * c_->h[2];
    // M = S^T W S, K = D^T W D on [0,1] (tensor.py tables), split into packed even/odd halves
    std::vector<double> M(N * N), K(N * N);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        double m = 0.0, k = 0.0;
        for (int q = 0; q < c_->nq; ++q) {
          m += c_->wq[q] * c_->S[q * N + i] * c_->S[q * N + j];
          k += c_->wq[q] * c_->D[q * N + i] * c_->D[q * N + j];
        }
        M[i * N + j] = m;
        K[i * N + j] = k;
      }
    // enforce the exact symmetries the packed storage assumes (they hold to rounding)
    auto symmetrise = [&](std::vector<double>& A) {
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          const double v = 0.25 * (A[i * N + j] + A[j * N + i] + A[(N - 1 - i) * N + (N - 1 - j)] +
                                   A[(N - 1 - j) * N + (N - 1 - i)]);
          A[i * N + j] = A[j * N + i] = A[(N - 1 - i) * N + (N - 1 - j)] = A[(N - 1 - j) * N + (N - 1 - i)] = v;
        }
    };
    symmetrise(M);
    symmetrise(K);
    constexpr int H = EOShape<N>::H, HE = EOShape<N>::HE;
    auto pack = [&](const std::vector<double>& A, T* Ae, T* Ao) {
      for (int i = 0; i < HE; ++i)
        for (int j = i; j < HE; ++j) {
          const bool mid = (N & 1) && (j == H);
          Ae[sym_idx(i, j)] = (T)(mid ? A[i * N + j] : 0.5 * (A[i * N + j] + A[i * N + (N - 1 - j)]));
        }
      for (int i = 0; i < H; ++i)
        for (int j = i; j < H; ++j) Ao[sym_idx(i, j)] = (T)(0.5 * (A[i * N + j] - A[i * N + (N - 1 - j)]));
    };
    pack(M, tab_.Me, tab_.Mo);
    for (int d = 0; d < 3; ++d) {
      const double gd = det / (c_->h[d] * c_->h[d]);
      tab_.g[d] = (T)gd;
      std::vector<double> Kd(K);
      for (double& v : Kd) v *= gd;
      pack(Kd, tab_.Ke[d], tab_.Ko[d]);
    }
    // separable factors of the GL-collocation diagonal (index 0: sum over the two cells at a cell boundary)
    for (int i = 0; i < P; ++i) {
      double dd0 = 0.0, ddp = 0.0, ddi = 0.0;
      for (int q = 0; q < N; ++q) {
        dd0 += c_->glw[q] * c_->glD[q * N + 0] * c_->glD[q * N + 0];
        ddp += c_->glw[q] * c_->glD[q * N + P] * c_->glD[q * N + P];
        ddi += c_->glw[q] * c_->glD[q * N + i] * c_->glD[q * N + i];
      }
      tab_.wa[i] = i == 0 ? c_->glw[0] + c_->glw[P] : c_->glw[i];
      tab_.da[i] = i == 0 ? dd0 + ddp : ddi;
    }
    tab_.wa[P] = tab_.da[P] = 0.0;
    tab_.diag_onfly = 0;
    general_ = c_->geometry != MFCG_GEOM_AFFINE;
    // curved mesh with more quadrature points than nodes per direction (BP3 / BP4 of the reference, n_q = p+2):
    // the cell-by-cell path (mfcg_cellpath.cuh); merged solves then run pre / apply / post as three kernels
    cellpath_ = general_ && c_->nq != N;
    if (cellpath_) {
      for (int q = 0; q < c_->nq; ++q)
        for (int i = 0; i < N; ++i) { ctab_.S[q * N + i] = c_->S[q * N + i]; ctab_.D[q * N + i] = c_->D[q * N + i]; }
      ctab_.n = N;
      ctab_.nq = c_->nq;
      cell_smem_ = (int)(sizeof(T) * 6 * c_->nq * c_->nq * c_->nq + sizeof(int) * N * N * N);
      MFCG_CUDA(cudaFuncSetAttribute(k_cell_general<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, cell_smem_));
      smem_ = cell_smem_;
      int rc = build_general_tables();
      if (rc) return rc;
    } else if (general_) {
      smem_ = (int)Geo<P, 1>::template smem_bytes<T>();
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 0, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 1, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      int rc = build_general_tables();
      if (rc) return rc;
    } else {
      smem_ = (int)Geo<P, 0>::template smem_bytes<T>();
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      MFCG_CUDA(cudaFuncSetAttribute(k_brick<P, T, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      if constexpr (Brick2Enabled<P>::value) {
        // the persistent TMA-fed kernel of the merged iteration (mfcg_brick2.cuh); MFCG_BRICK2=0 keeps the
        // first-generation kernel for comparisons
        const char* env = std::getenv("MFCG_BRICK2");
        brick2_ok_ = !(env && env[0] == '0');
        if (brick2_ok_)
          MFCG_CUDA(cudaFuncSetAttribute(k_brick2<P, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Geo2<P, T>::SMEM));
      }
    }
    vgrid_ = c_->ctx->sm_count * 8;
    if (const char* env = std::getenv("MFCG_COMP_INTERLEAVE")) comp_interleave_ = env[0] != '0';
    // one scalar field per component, fields 256-byte aligned; the gaps stay zero
    C_ = c_->ncomp;
    cs_ = C_ == 1 ? c_->grid.n_dofs : (c_->grid.n_dofs + 31) / 32 * 32;
    nt_ = cs_ * C_;
    rows_pc_ = c_->n_bricks + vgrid_;
    const i64 rows = rows_pc_ * C_;
    MFCG_CUDA(cudaMalloc(&partials_a_, sizeof(double) * 8 * rows));
    MFCG_CUDA(cudaMalloc(&partials_b_, sizeof(double) * 8 * rows));
    MFCG_CUDA(cudaMemsetAsync(partials_a_, 0, sizeof(double) * 8 * rows, stream()));
    MFCG_CUDA(cudaMemsetAsync(partials_b_, 0, sizeof(double) * 8 * rows, stream()));
    return MFCG_OK;
  }

  void info(mfcg_op_info* out) override {
    out->n_dofs = c_->grid.n_dofs * C_;
    out->n_interior = c_->grid.n_int;
    out->n_bricks = c_->n_bricks;
    for (int d = 0; d < 3; ++d) out->brick[d] = c_->grid.B[d];
    out->threads = general_ ? Cfg<P, 1>::THREADS : Cfg<P, 0>::THREADS;
    out->smem_bytes = smem_;
    if constexpr (Brick2Enabled<P>::value)
      if (brick2_ok_) { out->threads = Geo2<P, T>::THREADS; out->smem_bytes = (int)Geo2<P, T>::SMEM; }
    out->geometry_bytes = geo_bytes_;
  }

  int apply(const double* src, double* dst, int location) override {
    int rc = ensure_vectors(false);
    if (rc) return rc;
    if ((rc = load_vec(src, location, p_))) return rc;
    if ((rc = launch_apply(p_, v_))) return rc;
    if ((rc = store_vec(v_, dst, location))) return rc;
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    return MFCG_OK;
  }

  int diagonal(double* out, int location) override {
    int rc = ensure_diagonal();
    if (rc) return rc;
    const i64 n = c_->grid.n_dofs;
    double* target = location ? out : c_->d_io;
    k_to_user_order<double><<<vgrid_, VT, 0, stream()>>>(n, 1, n, c_->d_perm, c_->d_invdiag, target);
    MFCG_CUDA(cudaGetLastError());
    if (!location) MFCG_CUDA(cudaMemcpyAsync(out, c_->d_io, sizeof(double) * n, cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    return MFCG_OK;
  }

  int solve(const mfcg_solve_args* a, mfcg_solve_result* res) override;

  // copies the device-built table back as fp64: kind 1 final tensor, kind 2 inverse Jacobian then jxw
  int geometry(int kind, double* out_host, i64 n_doubles) override {
    if (!general_ || kind != c_->geometry || (kind != 1 && kind != 2)) {
      set_error("the operator holds no stored geometry table of that kind");
      return MFCG_EINVAL;
    }
    const i64 nq3 = (i64)c_->nq * c_->nq * c_->nq, nc = c_->n_cells;
    const i64 need = kind == 1 ? nc * nq3 * 6 : nc * nq3 * 10;
    if (n_doubles < need) { set_error("output buffer too small"); return MFCG_EINVAL; }
    const i64 na = kind == 1 ? nc * nq3 * 6 : nc * nq3 * 9;
    std::vector<T> tmp((size_t)std::max(na, nc * nq3));
    MFCG_CUDA(cudaMemcpy(tmp.data(), geo_a_, sizeof(T) * na, cudaMemcpyDeviceToHost));
    for (i64 i = 0; i < na; ++i) out_host[i] = (double)tmp[(size_t)i];
    if (kind == 2) {
      MFCG_CUDA(cudaMemcpy(tmp.data(), geo_b_, sizeof(T) * nc * nq3, cudaMemcpyDeviceToHost));
      for (i64 i = 0; i < nc * nq3; ++i) out_host[na + i] = (double)tmp[(size_t)i];
    }
    return MFCG_OK;
  }

 private:
  cudaStream_t stream() const { return c_->ctx->stream; }

  int ensure_vectors(bool all) {
    // +32 bytes: the brick kernel reads whole aligned 16-byte chunks
    auto need = [&](T** v) -> int {
      if (*v) return MFCG_OK;
      MFCG_CUDA(cudaMalloc(v, sizeof(T) * nt_ + 32));
      if (C_ > 1) MFCG_CUDA(cudaMemsetAsync(*v, 0, sizeof(T) * nt_ + 32, stream()));
      return MFCG_OK;
    };
    for (T** v : {&p_, &v_}) if (int rc = need(v)) return rc;
    if (all)
      for (T** v : {&x_, &r_, &z_, &minv_}) if (int rc = need(v)) return rc;
    return MFCG_OK;
  }

  // local assembly of the (uninverted) diagonal into diag (brick numbering, fp64)
  int assemble_diagonal(double* diag) {
    const i64 n = c_->grid.n_dofs;
    MFCG_CUDA(cudaMemsetAsync(diag, 0, sizeof(double) * n, stream()));
    MFCG_CUDA(cudaMemsetAsync(c_->d_flag, 0, sizeof(int), stream()));
    if (!general_) {
      DiagTables t{};
      for (int i = 0; i < N; ++i) {
        t.w[i] = c_->glw[i];
        double dd = 0.0;
        for (int q = 0; q < N; ++q) dd += c_->glw[q] * c_->glD[q * N + i] * c_->glD[q * N + i];
        t.dd[i] = dd;
      }
      const double det = c_->h[0] * c_->h[1] * c_->h[2];
      for (int d = 0; d < 3; ++d) t.g[d] = det / (c_->h[d] * c_->h[d]);
      k_diag_affine<<<vgrid_, VT, 0, stream()>>>(c_->grid, t, c_->n_cells, diag);
    } else {
      DiagGen dg{};
      for (int q = 0; q < N; ++q)
        for (int i = 0; i < N; ++i) dg.D2[q * N + i] = c_->glD[q * N + i] * c_->glD[q * N + i];
      for (int i = 0; i < N; ++i) dg.dd[i] = c_->glD[i * N + i];
      const PointTab pt = point_table(c_->glx, c_->glw);
      const size_t sm = sizeof(double) * 6 * N * N * N;
      k_diag_general<<<vgrid_, 128, sm, stream()>>>(c_->grid, geo_mesh(), pt, dg, c_->n_cells, diag, c_->d_flag);
    }
    MFCG_CUDA(cudaGetLastError());
    int gflag = 0;
    MFCG_CUDA(cudaMemcpyAsync(&gflag, c_->d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    if (gflag) { set_error("degenerate cell: det J <= 0"); return MFCG_EINVAL; }
    return MFCG_OK;
  }

  // diag -> 1/diag (constrained entries 1); takes ownership of diag on success
  int invert_diagonal(double* diag) {
    MFCG_CUDA(cudaMemsetAsync(c_->d_flag, 0, sizeof(int), stream()));
    k_diag_invert<<<vgrid_, VT, 0, stream()>>>(c_->grid, diag, c_->d_flag);
    MFCG_CUDA(cudaGetLastError());
    int flag = 0;
    MFCG_CUDA(cudaMemcpyAsync(&flag, c_->d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    if (flag) { set_error("operator diagonal is not positive definite"); return MFCG_EINVAL; }
    c_->d_invdiag = diag;
    return MFCG_OK;
  }

  int ensure_diagonal() {
    if (c_->d_invdiag) return MFCG_OK;
    if (c_->has_lower || c_->has_upper) {
      set_error("a slab operator needs its neighbours for the diagonal: use the slab-group entry points");
      return MFCG_EINVAL;
    }
    double* diag = nullptr;
    MFCG_CUDA(cudaMalloc(&diag, sizeof(double) * c_->grid.n_dofs));
    int rc = assemble_diagonal(diag);
    if (!rc) rc = invert_diagonal(diag);
    if (rc) cudaFree(diag);
    return rc;
  }

  // caller numbering (fp64, host or device) -> brick numbering (T, device)
  // `usr_comp` == 1: a per-node scalar replicated into every component field
  int load_vec(const double* usr, int location, T* dev, int usr_comp = 0) {
    const i64 n = c_->grid.n_dofs;
    if (usr_comp == 0) usr_comp = C_;
    const double* from = usr;
    if (!location) {
      MFCG_CUDA(cudaMemcpyAsync(c_->d_io, usr, sizeof(double) * n * usr_comp, cudaMemcpyHostToDevice, stream()));
      from = c_->d_io;
    }
    k_to_device_order<T><<<vgrid_, VT, 0, stream()>>>(n, C_, cs_, usr_comp, c_->d_perm, from, dev);
    MFCG_CUDA(cudaGetLastError());
    ++launches_;
    return MFCG_OK;
  }

  int store_vec(const T* dev, double* usr, int location) {
    const i64 n = c_->grid.n_dofs;
    double* target = location ? usr : c_->d_io;
    k_to_user_order<T><<<vgrid_, VT, 0, stream()>>>(n, C_, cs_, c_->d_perm, dev, target);
    MFCG_CUDA(cudaGetLastError());
    ++launches_;
    if (!location) MFCG_CUDA(cudaMemcpyAsync(usr, c_->d_io, sizeof(double) * n * C_, cudaMemcpyDeviceToHost, stream()));
    return MFCG_OK;
  }

  int launch_brick(int mode, const T* src, T* pv, T* v, double* partials, i64 first = 0, i64 count = -1) {
    if (count < 0) count = c_->n_bricks - first;
    if (count == 0) return MFCG_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (time_kernels_) {
      if (event_cursor_ + 2 > events_.size())
        for (int i = 0; i < 2; ++i) {
          cudaEvent_t e;
          MFCG_CUDA(cudaEventCreate(&e));
          events_.push_back(e);
        }
      e0 = events_[event_cursor_++];
      e1 = events_[event_cursor_++];
      MFCG_CUDA(cudaEventRecord(e0, stream()));
    }
    const unsigned nb = (unsigned)count;
    const int off = (int)first;
    // Several components on stored geometry go out as ONE launch with the blocks of a brick next to each other
    // (block = brick * C + component): the brick's geometry -- the largest stream of these kernels -- crosses HBM
    // once and is served from L2 to the other components.  MFCG_COMP_INTERLEAVE=0: one launch per component.
    if (C_ > 1 && general_ && !cellpath_ && c_->geometry != MFCG_GEOM_QUADRATIC_COMPUTE && comp_interleave_) {
      const i64 ps = 8 * rows_pc_;
      if (mode == 0)
        k_brick<P, T, 0, 1, true><<<nb * C_, Cfg<P, 1>::THREADS, smem_, stream()>>>(
            c_->grid, tab_, gen_, geo_, src, nullptr, v, nullptr, nullptr, nullptr, nullptr, nullptr, off, C_, cs_, ps);
      else
        k_brick<P, T, 1, 1, true><<<nb * C_, Cfg<P, 1>::THREADS, smem_, stream()>>>(
            c_->grid, tab_, gen_, geo_, nullptr, pv, v, r_, x_, minv_, c_->d_state, partials, off, C_, cs_, ps);
    } else
    for (int comp = 0; comp < C_; ++comp) {
      const i64 o = comp * cs_;
      const T* s_ = src ? src + o : nullptr;
      T* pv_ = pv ? pv + o : nullptr;
      T* vv_ = v + o;
      T *rr_ = r_ ? r_ + o : nullptr, *xx_ = x_ ? x_ + o : nullptr, *mm_ = minv_ ? minv_ + o : nullptr;
      double* part_ = partials ? partials + 8 * comp * rows_pc_ : nullptr;
      if (cellpath_) {
        if (mode != 0) { set_error("internal error: the cell path has no fused iteration"); return MFCG_ECUDA; }
        const unsigned cgrid = (unsigned)std::min<i64>(c_->n_cells, (i64)c_->ctx->sm_count * 16);
        k_cell_general<T><<<cgrid, 128, cell_smem_, stream()>>>(c_->grid, ctab_, geo_, qpt_, c_->n_cells, s_, vv_);
      } else if (!general_) {
        if (mode == 0)
          k_brick<P, T, 0, 0><<<nb, Cfg<P, 0>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, s_, nullptr, vv_, nullptr, nullptr, nullptr, nullptr, nullptr, off);
        else if (use_brick2_) {
          if constexpr (Brick2Enabled<P>::value) {
            const unsigned grid2 = std::min<unsigned>(nb, (unsigned)c_->ctx->sm_count);
            k_brick2<P, T><<<grid2, Geo2<P, T>::THREADS, Geo2<P, T>::SMEM, stream()>>>(
                c_->grid, tab_, tab_.diag_onfly ? 1 : 2, pv_, vv_, rr_, xx_, c_->d_state, part_, off, (int)nb);
          }
        } else
          k_brick<P, T, 1, 0><<<nb, Cfg<P, 0>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, nullptr, pv_, vv_, rr_, xx_, mm_, c_->d_state, part_, off);
      } else if (c_->geometry != MFCG_GEOM_QUADRATIC_COMPUTE) {
        if (mode == 0)
          k_brick<P, T, 0, 1><<<nb, Cfg<P, 1>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, s_, nullptr, vv_, nullptr, nullptr, nullptr, nullptr, nullptr, off);
        else
          k_brick<P, T, 1, 1><<<nb, Cfg<P, 1>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, nullptr, pv_, vv_, rr_, xx_, mm_, c_->d_state, part_, off);
      } else {
        if (mode == 0)
          k_brick<P, T, 0, 2><<<nb, Cfg<P, 2>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, s_, nullptr, vv_, nullptr, nullptr, nullptr, nullptr, nullptr, off);
        else
          k_brick<P, T, 1, 2><<<nb, Cfg<P, 2>::THREADS, smem_, stream()>>>(
              c_->grid, tab_, gen_, geo_, nullptr, pv_, vv_, rr_, xx_, mm_, c_->d_state, part_, off);
      }
    }
    MFCG_CUDA(cudaGetLastError());
    if (time_kernels_) MFCG_CUDA(cudaEventRecord(e1, stream()));
    ++launches_;
    ++op_launches_;
    return MFCG_OK;
  }

  // dst = A src in brick numbering
  int launch_apply(const T* src, T* dst) {
    const bool has_shared = c_->grid.n_dofs > c_->grid.n_int;
    if (cellpath_) {  // every DoF is accumulated atomically
      MFCG_CUDA(cudaMemsetAsync(dst, 0, sizeof(T) * nt_, stream()));
    } else if (has_shared) {
      for (int comp = 0; comp < C_; ++comp) k_surface_init<T><<<vgrid_, VT, 0, stream()>>>(c_->grid, dst + comp * cs_);
      MFCG_CUDA(cudaGetLastError());
      launches_ += C_;
    }
    int rc = launch_brick(0, src, nullptr, dst, nullptr);
    if (rc) return rc;
    if (has_shared) {
      for (int comp = 0; comp < C_; ++comp)
        k_surface_fix<T><<<vgrid_, VT, 0, stream()>>>(c_->grid, src + comp * cs_, dst + comp * cs_);
      MFCG_CUDA(cudaGetLastError());
      launches_ += C_;
    }
    return MFCG_OK;
  }

  // ------------------------------------------------------------------ slab group interface
 public:
  int g_alloc() override {
    if (cellpath_) { set_error("z-slabs of curved operators with n_q_1d > p+1 are not supported"); return MFCG_EUNSUPPORTED; }
    const i64 nxy = (i64)(c_->grid.cells[0] * P + 1) * (c_->grid.cells[1] * P + 1);
    for (int side = 0; side < 2; ++side)
      for (int rv = 0; rv < 2; ++rv)
        if (!plane_[side][rv]) MFCG_CUDA(cudaMalloc(&plane_[side][rv], sizeof(double) * nxy * C_));
    if (!d_sums_) MFCG_CUDA(cudaMalloc(&d_sums_, sizeof(double) * 8));
    if (!ev_front_) MFCG_CUDA(cudaEventCreateWithFlags(&ev_front_, cudaEventDisableTiming));
    return ensure_vectors(true);
  }
  bool g_has_diag() override { return c_->d_invdiag != nullptr; }
  void* g_plane(int side, int recv) override { return plane_[side][recv]; }
  size_t g_plane_bytes(bool diag_planes) override {
    const size_t nxy = (size_t)(c_->grid.cells[0] * P + 1) * (c_->grid.cells[1] * P + 1);
    return nxy * (diag_planes ? sizeof(double) : sizeof(T) * (size_t)C_);  // the diagonal is one value per node
  }
  double* g_sums() override { return d_sums_; }

  int g_diag_local() override {
    if (!diag_raw_) MFCG_CUDA(cudaMalloc(&diag_raw_, sizeof(double) * c_->grid.n_dofs));
    return assemble_diagonal(diag_raw_);
  }
  int g_diag_finish() override {
    double* d = diag_raw_;
    diag_raw_ = nullptr;
    int rc = invert_diagonal(d);
    if (rc) cudaFree(d);
    return rc;
  }

  // dst = A src on a slab: everything up to the hand-over of the interface planes
  int g_apply_front(const double* src, int location) override {
    int rc = g_alloc();
    if (rc) return rc;
    if ((rc = load_vec(src, location, p_))) return rc;
    const BrickGrid& g = c_->grid;
    const i64 nb = c_->n_bricks, nxy = (i64)g.mb[0] * g.mb[1];
    if (g.n_dofs > g.n_int) {
      for (int c = 0; c < C_; ++c) k_surface_init<T><<<vgrid_, VT, 0, stream()>>>(g, v_ + c * cs_);
      launches_ += C_;
    }
    if ((rc = launch_interface_first(0, p_, nullptr, v_, nullptr))) return rc;
    MFCG_CUDA(cudaStreamWaitEvent(c_->ctx->comm_stream, ev_front_, 0));
    return pack_planes(false);
  }
  int g_apply_end(double* dst, int location) override {
    const BrickGrid& g = c_->grid;
    if (g.n_dofs > g.n_int) {
      for (int c = 0; c < C_; ++c) k_surface_fix<T><<<vgrid_, VT, 0, stream()>>>(g, p_ + c * cs_, v_ + c * cs_);
      launches_ += C_;
    }
    int rc = store_vec(v_, dst, location);
    if (rc) return rc;
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    return MFCG_OK;
  }

  // Brick launches of a slab: the brick layers that touch an interface plane first (one launch: the top layer, then,
  // wrapping around the end of the brick list, the bottom layer), the event that releases the communication
  // stream, then the rest.  A slab without neighbours, or of at most two brick layers, goes out as one launch.
  int launch_interface_first(int mode, const T* src, T* pv, T* v, double* partials) {
    const BrickGrid& g = c_->grid;
    const i64 nb = c_->n_bricks, nxy = (i64)g.mb[0] * g.mb[1];
    const bool lo = c_->has_lower, hi = c_->has_upper;
    int rc;
    if (g.mb[2] <= 2 || (!lo && !hi)) {
      if ((rc = launch_brick(mode, src, pv, v, partials))) return rc;
      MFCG_CUDA(cudaEventRecord(ev_front_, stream()));
      return MFCG_OK;
    }
    const i64 first = hi ? nb - nxy : 0, count = (lo && hi) ? 2 * nxy : nxy;
    if ((rc = launch_brick(mode, src, pv, v, partials, first, count))) return rc;
    MFCG_CUDA(cudaEventRecord(ev_front_, stream()));
    const i64 rest_first = lo ? nxy : 0;   // interior layers (+ the far layer of a slab with one neighbour)
    return launch_brick(mode, src, pv, v, partials, rest_first, nb - count);
  }

  // pack the interface planes of v (or of the raw diagonal) on the communication stream
  int pack_planes(bool diag_planes) {
    cudaStream_t cs = c_->ctx->comm_stream;
    const int Ktop = c_->grid.cells[2] * P;
    const i64 nxy = (i64)(c_->grid.cells[0] * P + 1) * (c_->grid.cells[1] * P + 1);
    for (int side = 0; side < 2; ++side) {
      if (!(side == 0 ? c_->has_lower : c_->has_upper)) continue;
      const int K = side == 0 ? 0 : Ktop;
      if (diag_planes) {
        k_plane_pack<double><<<vgrid_, VT, 0, cs>>>(c_->grid, K, diag_raw_, (double*)plane_[side][0]);
        ++launches_;
      } else {
        for (int c = 0; c < C_; ++c)  // component fields one after the other in the plane buffer
          k_plane_pack<T><<<vgrid_, VT, 0, cs>>>(c_->grid, K, v_ + c * cs_, (T*)plane_[side][0] + c * nxy);
        launches_ += C_;
      }
    }
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  // one merged iteration up to the hand-over of the interface planes: pre on shared DoFs, the
  // brick layers touching the interface first, then (event) the interior layers on the compute
  // stream while the planes are packed on the communication stream
  int g_front(bool diag_planes) override {
    cudaStream_t cs = c_->ctx->comm_stream;
    if (diag_planes) {
      MFCG_CUDA(cudaEventRecord(ev_front_, stream()));
      MFCG_CUDA(cudaStreamWaitEvent(cs, ev_front_, 0));
      return pack_planes(true);
    }
    const BrickGrid& g = c_->grid;
    const i64 n = g.n_dofs, nb = c_->n_bricks, nxy = (i64)g.mb[0] * g.mb[1];
    if (n > g.n_int) {
      for (int c = 0; c < C_; ++c) {
        const i64 o = c * cs_;
        k_pre<T><<<vgrid_, VT, 0, stream()>>>(g, g.n_int, n, 1, r_ + o, p_ + o, v_ + o, x_ + o, minv_ + o, c_->d_state);
      }
      launches_ += C_;
    }
    int rc;
    if ((rc = launch_interface_first(1, nullptr, p_, v_, partials_a_))) return rc;
    MFCG_CUDA(cudaStreamWaitEvent(cs, ev_front_, 0));
    return pack_planes(false);
  }

  // add the neighbours' contributions (communication stream)
  int g_unpack(bool diag_planes) override {
    cudaStream_t cs = c_->ctx->comm_stream;
    const int Ktop = c_->grid.cells[2] * P;
    const i64 nxy = (i64)(c_->grid.cells[0] * P + 1) * (c_->grid.cells[1] * P + 1);
    for (int side = 0; side < 2; ++side) {
      if (!(side == 0 ? c_->has_lower : c_->has_upper)) continue;
      const int K = side == 0 ? 0 : Ktop;
      if (diag_planes) {
        k_plane_add<double><<<vgrid_, VT, 0, cs>>>(c_->grid, K, diag_raw_, (const double*)plane_[side][1]);
        ++launches_;
      } else {
        for (int c = 0; c < C_; ++c)
          k_plane_add<T><<<vgrid_, VT, 0, cs>>>(c_->grid, K, v_ + c * cs_, (const T*)plane_[side][1] + c * nxy);
        launches_ += C_;
      }
    }
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  // post on the shared range (ghost plane excluded) and the slab's seven sums
  int g_post() override {
    const BrickGrid& g = c_->grid;
    const i64 n = g.n_dofs;
    // rows of partial sums: per component, one per brick and one per k_post block (unused rows stay zero)
    const int rows = (int)(rows_pc_ * C_);
    if (n > g.n_int) {
      for (int c = 0; c < C_; ++c) {
        const i64 o = c * cs_;
        k_post<T><<<vgrid_, VT, 0, stream()>>>(g, g.n_int, n, 1, r_ + o, p_ + o, v_ + o, minv_ + o, c_->d_state,
                                               partials_a_ + 8 * (c * rows_pc_ + c_->n_bricks));
      }
      launches_ += C_;
    }
    k_reduce_partials<<<1, 256, 0, stream()>>>(partials_a_, rows, 7, 0, d_sums_);
    ++launches_;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  int g_scalar(const double* global_sums_dev) override {
    k_scalar_merged_sums<<<1, 32, 0, stream()>>>(global_sums_dev, c_->d_state, d_history_);
    ++launches_;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  int g_poll(int* active) override {
    MFCG_CUDA(cudaMemcpyAsync(c_->h_state, c_->d_state, sizeof(SolveState), cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    *active = c_->h_state->active;
    return MFCG_OK;
  }

  // a.b over the DoFs this slab owns, all components -> out[0]
  int dot_owned(const T* a, const T* b, double* partials, double* out) {
    for (int c = 0; c < C_; ++c)
      k_dot_owned<T><<<vgrid_, VT, 0, stream()>>>(c_->grid, a + c * cs_, b + c * cs_, partials + 8 * (i64)c * vgrid_);
    k_reduce_partials<<<1, 256, 0, stream()>>>(partials, vgrid_ * C_, 1, 0, out);
    launches_ += C_ + 1;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  // right-hand side, preconditioner, zero vectors, this slab's part of b.b
  int g_begin(const mfcg_solve_args* a, int limit) override {
    const i64 n = c_->grid.n_dofs;
    int rc = g_alloc();
    if (rc) return rc;
    if (history_cap_ < limit) {
      if (d_history_) cudaFree(d_history_);
      MFCG_CUDA(cudaMalloc(&d_history_, sizeof(double) * 4 * (size_t)limit));
      history_cap_ = limit;
    }
    launches_ = op_launches_ = 0;
    time_kernels_ = false;
    event_cursor_ = 0;
    if ((rc = load_vec(a->b, a->location, r_))) return rc;
    const bool prec = a->variant == MFCG_COMBINED_PCG;
    tab_.diag_onfly = (prec && !a->inv_diag && !general_) ? 1 : 0;
    use_brick2_ = brick2_ok_ && (tab_.diag_onfly || !prec);
    if (prec) {
      if (a->inv_diag) {  // one value per node (solvers.py:617-621), replicated into the component fields
        if ((rc = load_vec(a->inv_diag, a->location, minv_, 1))) return rc;
      } else {
        for (int c = 0; c < C_; ++c) k_convert<T, double><<<vgrid_, VT, 0, stream()>>>(n, c_->d_invdiag, minv_ + c * cs_);
        launches_ += C_;
      }
    } else {
      k_fill<T><<<vgrid_, VT, 0, stream()>>>(nt_, minv_, (T)1);
      ++launches_;
    }
    MFCG_CUDA(cudaMemsetAsync(x_, 0, sizeof(T) * nt_, stream()));
    MFCG_CUDA(cudaMemsetAsync(p_, 0, sizeof(T) * nt_, stream()));
    MFCG_CUDA(cudaMemsetAsync(v_, 0, sizeof(T) * nt_, stream()));
    if ((rc = dot_owned(r_, r_, partials_a_, d_sums_))) return rc;
    // rows no kernel of the iteration writes must read as zero in g_post
    MFCG_CUDA(cudaMemsetAsync(partials_a_, 0, sizeof(double) * 8 * rows_pc_ * C_, stream()));
    return MFCG_OK;
  }

  int g_set_state(const mfcg_solve_args* a, int limit, const double* global_bb_dev) override {
    SolveState s0;
    std::memset(&s0, 0, sizeof(s0));
    s0.active = 1;
    s0.fixed = a->fixed_iterations >= 0 ? 1 : 0;
    s0.force_x = a->force_x_updates ? 1 : 0;
    s0.has_prec = (a->variant == MFCG_COMBINED_PCG || a->variant == MFCG_PCG) ? 1 : 0;
    s0.limit = limit;
    s0.tol = a->tolerance;
    s0.residual = 1.0;
    *c_->h_state = s0;
    MFCG_CUDA(cudaMemcpyAsync(c_->d_state, c_->h_state, sizeof(SolveState), cudaMemcpyHostToDevice, stream()));
    k_set_bnorm<<<1, 1, 0, stream()>>>(c_->d_state, global_bb_dev);
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  // ---- standard (P)CG on a slab (BASELINE configs[3]/[4] arm "standard vs merged")
  int g_std_begin(const mfcg_solve_args* a, int limit) override {
    const i64 n = c_->grid.n_dofs;
    int rc = g_alloc();
    if (rc) return rc;
    if (history_cap_ < limit) {
      if (d_history_) cudaFree(d_history_);
      MFCG_CUDA(cudaMalloc(&d_history_, sizeof(double) * 4 * (size_t)limit));
      history_cap_ = limit;
    }
    launches_ = op_launches_ = 0;
    time_kernels_ = false;
    event_cursor_ = 0;
    use_brick2_ = false;
    tab_.diag_onfly = 0;
    std_prec_ = a->variant == MFCG_PCG;
    if ((rc = load_vec(a->b, a->location, v_))) return rc;   // b is staged in v, as in run_standard
    if (std_prec_) {
      if (a->inv_diag) {
        if ((rc = load_vec(a->inv_diag, a->location, minv_, 1))) return rc;
      } else {
        for (int c = 0; c < C_; ++c) k_convert<T, double><<<vgrid_, VT, 0, stream()>>>(n, c_->d_invdiag, minv_ + c * cs_);
        launches_ += C_;
      }
    }
    return dot_owned(v_, v_, partials_a_, d_sums_);   // b.b of this slab
  }
  // after g_set_state: r = b, z = M r, p = z, x = 0 and this slab's r.z, r.r
  int g_std_init_vectors() override {
    for (int c = 0; c < C_; ++c) {
      const i64 o = c * cs_;
      k_std_init_owned<T><<<vgrid_, VT, 0, stream()>>>(c_->grid, v_ + o, std_prec_ ? minv_ + o : nullptr, r_ + o, z_ + o,
                                                       p_ + o, x_ + o, partials_a_ + 8 * (i64)c * vgrid_);
    }
    k_reduce_partials<<<1, 256, 0, stream()>>>(partials_a_, vgrid_ * C_, 2, 0, d_sums_);
    launches_ += C_ + 1;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }
  int g_std_init_scalar(const double* global_sums_dev) override {
    k_std_init_scalar<<<1, 256, 0, stream()>>>(global_sums_dev, 1, c_->d_state);  // one row: r.z, r.r
    ++launches_;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }
  int g_std_apply_front() override {
    const BrickGrid& g = c_->grid;
    const i64 nb = c_->n_bricks, nxy = (i64)g.mb[0] * g.mb[1];
    int rc;
    if (g.n_dofs > g.n_int) {
      for (int c = 0; c < C_; ++c) k_surface_init<T><<<vgrid_, VT, 0, stream()>>>(g, v_ + c * cs_);
      launches_ += C_;
    }
    if ((rc = launch_interface_first(0, p_, nullptr, v_, nullptr))) return rc;
    MFCG_CUDA(cudaStreamWaitEvent(c_->ctx->comm_stream, ev_front_, 0));
    return pack_planes(false);
  }
  int g_std_apply_end() override {
    const BrickGrid& g = c_->grid;
    if (g.n_dofs > g.n_int) {
      for (int c = 0; c < C_; ++c) k_surface_fix<T><<<vgrid_, VT, 0, stream()>>>(g, p_ + c * cs_, v_ + c * cs_);
      launches_ += C_;
    }
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }
  int g_std_dot_pv() override { return dot_owned(p_, v_, partials_a_, d_sums_); }
  int g_std_alpha_update(const double* global_sums_dev) override {
    const i64 n = nt_;  // flat over the component fields
    k_std_alpha<<<1, 256, 0, stream()>>>(global_sums_dev, 1, c_->d_state);
    k_std_axpy<T><<<vgrid_, VT, 0, stream()>>>(n, x_, p_, 1.0, c_->d_state);
    k_std_axpy<T><<<vgrid_, VT, 0, stream()>>>(n, r_, v_, -1.0, c_->d_state);
    launches_ += 3;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }
  // this slab's r.r (sum 0) and r.z (sum 1; = r.r without preconditioner)
  int g_std_dots_r() override {
    const i64 n = nt_;
    int rc = dot_owned(r_, r_, partials_a_, d_sums_);
    if (rc) return rc;
    if (std_prec_) {
      k_std_prec<T><<<vgrid_, VT, 0, stream()>>>(n, z_, minv_, r_, c_->d_state);
      ++launches_;
      if ((rc = dot_owned(r_, z_, partials_b_, d_sums_ + 1))) return rc;
    }
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }
  // global_sums_dev: row 0 = (r.r, r.z)
  int g_std_beta_p(const double* global_sums_dev) override {
    const i64 n = nt_;
    k_std_beta_sums<<<1, 32, 0, stream()>>>(global_sums_dev, std_prec_ ? 1 : 0, c_->d_state, d_history_);
    k_std_update_p<T><<<vgrid_, VT, 0, stream()>>>(n, p_, std_prec_ ? z_ : r_, c_->d_state);
    launches_ += 2;
    MFCG_CUDA(cudaGetLastError());
    return MFCG_OK;
  }

  int g_end(const mfcg_solve_args* a, mfcg_solve_result* res) override {
    std::memset(res, 0, sizeof(*res));
    const i64 n = c_->grid.n_dofs;
    if (a->variant == MFCG_COMBINED_CG || a->variant == MFCG_COMBINED_PCG) {  // x catch-up of the merged loop
      k_finalize_x<T><<<vgrid_, VT, 0, stream()>>>(nt_, x_, p_, r_, minv_, c_->d_state);
      ++launches_;
    }
    int rc = store_vec(x_, a->x, a->location);
    if (rc) return rc;
    MFCG_CUDA(cudaMemcpyAsync(c_->h_state, c_->d_state, sizeof(SolveState), cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    const SolveState& s = *c_->h_state;
    res->bnorm = s.bnorm;
    res->kernel_launches = launches_;
    res->operator_launches = op_launches_;
    res->iterations = s.k;
    res->matvecs = s.k;
    res->residual = s.residual;
    res->breakdown = s.breakdown;
    res->breakdown_iteration = s.breakdown_iteration;
    res->breakdown_value = s.breakdown_value;
    res->converged = a->fixed_iterations >= 0 ? (s.residual < a->tolerance) : s.converged;
    if (a->history && s.k > 0)
      MFCG_CUDA(cudaMemcpy(a->history, d_history_, sizeof(double) * 4 * (size_t)s.k, cudaMemcpyDeviceToHost));
    if (s.breakdown) {
      char buf[160];
      std::snprintf(buf, sizeof(buf), "breakdown code %d: value %.3e <= 0 at iteration %d", s.breakdown,
                    s.breakdown_value, s.breakdown_iteration);
      set_error(buf);
      return MFCG_EBREAKDOWN;
    }
    return MFCG_OK;
  }

 private:
  GeoMesh geo_mesh() const {
    GeoMesh gm{};
    for (int d = 0; d < 3; ++d) { gm.cells[d] = c_->grid.cells[d]; gm.h[d] = c_->h[d]; gm.ext[d] = c_->extents[d]; }
    gm.z0 = c_->slab_z0;
    gm.amp = c_->deformation;
    return gm;
  }

  // quadratic Lagrange basis on {0, 1/2, 1} and its derivative at 1D points t (mesh.py:150-170)
  static PointTab point_table(const std::vector<double>& t, const std::vector<double>& w) {
    PointTab pt{};
    pt.n = (int)t.size();
    for (int i = 0; i < pt.n; ++i) {
      const double x = t[i];
      pt.qv[3 * i + 0] = 2.0 * (x - 0.5) * (x - 1.0); pt.qv[3 * i + 1] = -4.0 * x * (x - 1.0); pt.qv[3 * i + 2] = 2.0 * x * (x - 0.5);
      pt.qd[3 * i + 0] = 4.0 * x - 3.0; pt.qd[3 * i + 1] = 4.0 - 8.0 * x; pt.qd[3 * i + 2] = 4.0 * x - 1.0;
      pt.w[i] = w[i];
    }
    return pt;
  }

  // halves of S and of the collocation derivative Dc, and the device geometry tables
  int build_general_tables() {
    constexpr int H = EOShape<N>::H, HE = EOShape<N>::HE;
    const std::vector<double>& S = c_->S;  // [q][i]
    if (!cellpath_) {  // even/odd halves of S and Dc for the brick kernels (n_q == N)
    // Dc[q][r]: derivative at x_q of the Lagrange polynomial through the quadrature points
    std::vector<double> Dc(N * N, 0.0);
    const std::vector<double>& x = c_->xq;
    for (int r = 0; r < N; ++r) {
      double wr = 1.0;
      for (int j = 0; j < N; ++j) if (j != r) wr /= (x[r] - x[j]);
      for (int q = 0; q < N; ++q) {
        double acc = 0.0;
        for (int m = 0; m < N; ++m) {
          if (m == r) continue;
          double prod = 1.0;
          for (int j = 0; j < N; ++j) if (j != r && j != m) prod *= (x[q] - x[j]);
          acc += prod;
        }
        Dc[q * N + r] = wr * acc;
      }
    }
    for (int q = 0; q < HE; ++q)
      for (int i = 0; i < HE; ++i) {
        const bool mid = (N & 1) && i == H;
        gen_.Se[q * HE + i] = (T)(mid ? S[q * N + i] : 0.5 * (S[q * N + i] + S[q * N + (N - 1 - i)]));
      }
    for (int q = 0; q < H; ++q)
      for (int i = 0; i < H; ++i) gen_.So[q * H + i] = (T)(0.5 * (S[q * N + i] - S[q * N + (N - 1 - i)]));
    for (int q = 0; q < H; ++q)
      for (int r = 0; r < HE; ++r) {
        const bool mid = (N & 1) && r == H;
        gen_.Be[q * HE + r] = (T)(mid ? Dc[q * N + r] : 0.5 * (Dc[q * N + r] + Dc[q * N + (N - 1 - r)]));
      }
    for (int q = 0; q < HE; ++q)
      for (int r = 0; r < H; ++r) gen_.Bo[q * H + r] = (T)(0.5 * (Dc[q * N + r] - Dc[q * N + (N - 1 - r)]));
    }
    const PointTab pt = point_table(c_->xq, c_->wq);
    if (!cellpath_)
      for (int i = 0; i < N; ++i) {
        for (int c = 0; c < 3; ++c) { gen_.qv[3 * i + c] = (T)pt.qv[3 * i + c]; gen_.qd[3 * i + c] = (T)pt.qd[3 * i + c]; }
        gen_.w3[i] = (T)c_->wq[i];
      }
    qpt_ = pt;
    const i64 nc = c_->n_cells, nq3 = (i64)c_->nq * c_->nq * c_->nq;
    const int kind = c_->geometry;
    double* nodes = nullptr;
    MFCG_CUDA(cudaMemsetAsync(c_->d_flag, 0, sizeof(int), stream()));
    if (kind == MFCG_GEOM_FINAL_TENSOR_LOAD) {
      geo_bytes_ = sizeof(T) * nc * nq3 * 6;
      MFCG_CUDA(cudaMalloc(&geo_a_, geo_bytes_));
    } else if (kind == MFCG_GEOM_INVERSE_JACOBIAN_LOAD) {
      geo_bytes_ = sizeof(T) * nc * nq3 * 10;
      MFCG_CUDA(cudaMalloc(&geo_a_, sizeof(T) * nc * nq3 * 9));
      MFCG_CUDA(cudaMalloc(&geo_b_, sizeof(T) * nc * nq3));
    } else {
      geo_bytes_ = sizeof(double) * nc * 81;
      MFCG_CUDA(cudaMalloc(&geo_a_, geo_bytes_));
      nodes = reinterpret_cast<double*>(geo_a_);
    }
    k_geometry<T><<<vgrid_from_ctx(), 128, 0, stream()>>>(geo_mesh(), pt, nc, kind, reinterpret_cast<T*>(geo_a_),
                                                          reinterpret_cast<T*>(geo_b_), nodes, c_->d_flag);
    MFCG_CUDA(cudaGetLastError());
    int flag = 0;
    MFCG_CUDA(cudaMemcpyAsync(&flag, c_->d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    if (flag) { set_error("degenerate cell: det J <= 0"); return MFCG_EINVAL; }
    geo_.kind = kind;
    geo_.data = geo_a_;
    geo_.jxw = geo_b_;
    return MFCG_OK;
  }
  int vgrid_from_ctx() const { return c_->ctx->sm_count * 8; }

  int run_merged(const mfcg_solve_args* a, int limit);
  int run_standard(const mfcg_solve_args* a, int limit, bool prec);

  OpCommon* c_;
  SepTables<T, N> tab_{};
  GenTables<T, N> gen_{};
  GeomAccess geo_{0, nullptr, nullptr};
  void* geo_a_ = nullptr;
  void* geo_b_ = nullptr;
  i64 geo_bytes_ = 0;
  bool comp_interleave_ = true;  // several components on stored geometry in one launch
  bool general_ = false;
  bool cellpath_ = false;  // curved mesh with n_q_1d != p+1: cell-by-cell apply
  CellTables ctab_{};
  PointTab qpt_{};
  int cell_smem_ = 0;
  bool brick2_ok_ = false, use_brick2_ = false;
  bool std_prec_ = false;  // slab-group standard solve: with Jacobi preconditioner
  void* plane_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [side lo/hi][send/recv]
  double* d_sums_ = nullptr;
  double* diag_raw_ = nullptr;  // slab runs: diagonal before the interface exchange
  cudaEvent_t ev_front_ = nullptr;
  int smem_ = 0, vgrid_ = 0;
  int C_ = 1;                         // components
  i64 cs_ = 0, nt_ = 0, rows_pc_ = 0;  // component stride, device vector length, partial rows per component
  T *x_ = nullptr, *r_ = nullptr, *p_ = nullptr, *v_ = nullptr, *z_ = nullptr, *minv_ = nullptr;
  double *partials_a_ = nullptr, *partials_b_ = nullptr, *d_history_ = nullptr;
  int history_cap_ = 0;
  std::vector<cudaEvent_t> events_;
  size_t event_cursor_ = 0;
  bool time_kernels_ = false;
  i64 launches_ = 0, op_launches_ = 0;
};

template <int P, typename T>
int Engine<P, T>::run_merged(const mfcg_solve_args* a, int limit) {
  const BrickGrid& g = c_->grid;
  const i64 n = g.n_dofs, n_sh = g.n_dofs - g.n_int;
  const bool fixed = a->fixed_iterations >= 0;
  // rows of partial sums: per component, one per brick and one per k_post block (unused rows stay zero)
  const int rows_fused = (int)(rows_pc_ * C_);
  const bool fused = a->fused && !cellpath_;
  for (int it = 1; it <= limit; ++it) {
    if (fused) {
      if (n_sh > 0) {
        for (int c = 0; c < C_; ++c) {
          const i64 o = c * cs_;
          k_pre<T><<<vgrid_, VT, 0, stream()>>>(g, g.n_int, n, 1, r_ + o, p_ + o, v_ + o, x_ + o, minv_ + o, c_->d_state);
        }
        launches_ += C_;
      }
      int rc = launch_brick(1, nullptr, p_, v_, partials_a_);
      if (rc) return rc;
      if (n_sh > 0) {
        for (int c = 0; c < C_; ++c) {
          const i64 o = c * cs_;
          k_post<T><<<vgrid_, VT, 0, stream()>>>(g, g.n_int, n, 1, r_ + o, p_ + o, v_ + o, minv_ + o, c_->d_state,
                                                 partials_a_ + 8 * (c * rows_pc_ + c_->n_bricks));
        }
        launches_ += C_;
      }
      k_scalar_merged<<<1, 256, 0, stream()>>>(partials_a_, rows_fused, c_->d_state, d_history_);
      ++launches_;
    } else {
      // the paper's GPU scheme: pre, mat-vec and post as separate kernels
      for (int c = 0; c < C_; ++c) {
        const i64 o = c * cs_;
        k_pre<T><<<vgrid_, VT, 0, stream()>>>(g, 0, n, 0, r_ + o, p_ + o, v_ + o, x_ + o, minv_ + o, c_->d_state);
      }
      int rc = launch_apply(p_, v_);
      if (rc) return rc;
      for (int c = 0; c < C_; ++c) {
        const i64 o = c * cs_;
        k_post<T><<<vgrid_, VT, 0, stream()>>>(g, 0, n, 0, r_ + o, p_ + o, v_ + o, minv_ + o, c_->d_state,
                                               partials_a_ + 8 * c * vgrid_);
      }
      k_scalar_merged<<<1, 256, 0, stream()>>>(partials_a_, vgrid_ * C_, c_->d_state, d_history_);
      launches_ += 2 * C_ + 1;
    }
    MFCG_CUDA(cudaGetLastError());
    if (!fixed && (it % 8 == 0)) {
      MFCG_CUDA(cudaMemcpyAsync(c_->h_state, c_->d_state, sizeof(SolveState), cudaMemcpyDeviceToHost, stream()));
      MFCG_CUDA(cudaStreamSynchronize(stream()));
      if (!c_->h_state->active) break;
    }
  }
  k_finalize_x<T><<<vgrid_, VT, 0, stream()>>>(nt_, x_, p_, r_, minv_, c_->d_state);
  MFCG_CUDA(cudaGetLastError());
  ++launches_;
  return MFCG_OK;
}

template <int P, typename T>
int Engine<P, T>::run_standard(const mfcg_solve_args* a, int limit, bool prec) {
  const BrickGrid& g = c_->grid;
  const i64 n = nt_;  // flat over all component fields
  const bool fixed = a->fixed_iterations >= 0;
  T* z = prec ? z_ : r_;
  // v_ holds b in brick numbering on entry
  k_std_init<T><<<vgrid_, VT, 0, stream()>>>(n, v_, prec ? minv_ : nullptr, r_, z_, p_, x_, partials_a_);
  k_std_init_scalar<<<1, 256, 0, stream()>>>(partials_a_, vgrid_, c_->d_state);
  launches_ += 2;
  MFCG_CUDA(cudaGetLastError());
  for (int it = 1; it <= limit; ++it) {
    int rc = launch_apply(p_, v_);
    if (rc) return rc;
    k_dot<T><<<vgrid_, VT, 0, stream()>>>(n, p_, v_, c_->d_state, partials_a_);
    k_std_alpha<<<1, 256, 0, stream()>>>(partials_a_, vgrid_, c_->d_state);
    k_std_axpy<T><<<vgrid_, VT, 0, stream()>>>(n, x_, p_, 1.0, c_->d_state);
    k_std_axpy<T><<<vgrid_, VT, 0, stream()>>>(n, r_, v_, -1.0, c_->d_state);
    k_dot<T><<<vgrid_, VT, 0, stream()>>>(n, r_, r_, c_->d_state, partials_a_);
    launches_ += 5;
    if (prec) {
      k_std_prec<T><<<vgrid_, VT, 0, stream()>>>(n, z_, minv_, r_, c_->d_state);
      k_dot<T><<<vgrid_, VT, 0, stream()>>>(n, r_, z_, c_->d_state, partials_b_);
      launches_ += 2;
    }
    k_std_beta<<<1, 256, 0, stream()>>>(partials_a_, prec ? partials_b_ : nullptr, vgrid_, c_->d_state, d_history_);
    k_std_update_p<T><<<vgrid_, VT, 0, stream()>>>(n, p_, z, c_->d_state);
    launches_ += 2;
    MFCG_CUDA(cudaGetLastError());
    if (!fixed && (it % 8 == 0)) {
      MFCG_CUDA(cudaMemcpyAsync(c_->h_state, c_->d_state, sizeof(SolveState), cudaMemcpyDeviceToHost, stream()));
      MFCG_CUDA(cudaStreamSynchronize(stream()));
      if (!c_->h_state->active) break;
    }
  }
  return MFCG_OK;
}

template <int P, typename T>
int Engine<P, T>::solve(const mfcg_solve_args* a, mfcg_solve_result* res) {
  std::memset(res, 0, sizeof(*res));
  const BrickGrid& g = c_->grid;
  const i64 n = nt_;  // flat over all component fields (gaps between fields are zero)
  const bool merged = a->variant == MFCG_COMBINED_CG || a->variant == MFCG_COMBINED_PCG;
  const bool prec = a->variant == MFCG_PCG || a->variant == MFCG_COMBINED_PCG;
  if (a->variant < 0 || a->variant > 3) { set_error("unknown solver variant"); return MFCG_EINVAL; }
  if (!a->b || !a->x) { set_error("b and x must not be NULL"); return MFCG_EINVAL; }
  if (a->tolerance <= 0) { set_error("tolerance must be positive"); return MFCG_EINVAL; }
  if (a->max_iterations < 1) { set_error("max_iterations must be at least 1"); return MFCG_EINVAL; }
  const bool fixed = a->fixed_iterations >= 0;
  // solvers.py:210: `limit = cfg.fixed_iterations or cfg.max_iterations` (0 falls through)
  const int limit = a->fixed_iterations > 0 ? a->fixed_iterations : a->max_iterations;
  int rc = ensure_vectors(true);
  if (rc) return rc;
  if (history_cap_ < limit) {
    if (d_history_) cudaFree(d_history_);
    MFCG_CUDA(cudaMalloc(&d_history_, sizeof(double) * 4 * (size_t)limit));
    history_cap_ = limit;
  }
  launches_ = op_launches_ = 0;
  time_kernels_ = a->time_kernels != 0;
  event_cursor_ = 0;

  EventPair ev;  // destroyed on every return path
  MFCG_CUDA(ev.create());
  cudaEvent_t t0 = ev.a, t1 = ev.b;
  MFCG_CUDA(cudaEventRecord(t0, stream()));

  // right-hand side: merged variants start with r = b, the standard ones stage b in v
  if ((rc = load_vec(a->b, a->location, merged ? r_ : v_))) return rc;
  // the operator's own Jacobi diagonal on an affine mesh is separable: interior DoFs compute it
  tab_.diag_onfly = (merged && prec && !a->inv_diag && !general_ && a->fused) ? 1 : 0;  // general_ covers the cell path
  // persistent kernel: 1/diag is either the operator's own (computed in the kernel) or the identity
  use_brick2_ = brick2_ok_ && merged && a->fused && (tab_.diag_onfly || !prec);
  if (prec) {
    if (a->inv_diag) {
      if ((rc = load_vec(a->inv_diag, a->location, minv_, 1))) return rc;
    } else {
      if ((rc = ensure_diagonal())) return rc;
      for (int c = 0; c < C_; ++c)
        k_convert<T, double><<<vgrid_, VT, 0, stream()>>>(g.n_dofs, c_->d_invdiag, minv_ + c * cs_);
      launches_ += C_;
    }
  } else if (merged) {
    k_fill<T><<<vgrid_, VT, 0, stream()>>>(n, minv_, (T)1);
    ++launches_;
  }
  const T* bvec = merged ? r_ : v_;
  k_dot<T><<<vgrid_, VT, 0, stream()>>>(n, bvec, bvec, nullptr, partials_a_);
  ++launches_;
  MFCG_CUDA(cudaGetLastError());
  std::vector<double> hp(8 * (size_t)vgrid_);
  MFCG_CUDA(cudaMemcpyAsync(hp.data(), partials_a_, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, stream()));
  MFCG_CUDA(cudaStreamSynchronize(stream()));
  double bb = 0.0;
  for (int i = 0; i < vgrid_; ++i) bb += hp[8 * (size_t)i];
  const double bnorm = std::sqrt(bb);
  res->bnorm = bnorm;
  if (bnorm == 0.0) {  // solvers.py:156-157, 191-192: zero rhs -> x = 0, 0 iterations, converged
    MFCG_CUDA(cudaMemsetAsync(x_, 0, sizeof(T) * n, stream()));
    if ((rc = store_vec(x_, a->x, a->location))) return rc;
    MFCG_CUDA(cudaStreamSynchronize(stream()));
    res->converged = 1;
    return MFCG_OK;
  }
  SolveState s0;
  std::memset(&s0, 0, sizeof(s0));
  s0.active = 1;
  s0.fixed = fixed ? 1 : 0;
  s0.force_x = a->force_x_updates ? 1 : 0;
  s0.has_prec = prec ? 1 : 0;
  s0.limit = limit;
  s0.bnorm = bnorm;
  s0.tol = a->tolerance;
  s0.residual = 1.0;  // ||r0|| / ||b|| with r0 = b
  *c_->h_state = s0;
  MFCG_CUDA(cudaMemcpyAsync(c_->d_state, c_->h_state, sizeof(SolveState), cudaMemcpyHostToDevice, stream()));
  if (merged) {
    MFCG_CUDA(cudaMemsetAsync(x_, 0, sizeof(T) * n, stream()));
    MFCG_CUDA(cudaMemsetAsync(p_, 0, sizeof(T) * n, stream()));
    MFCG_CUDA(cudaMemsetAsync(v_, 0, sizeof(T) * n, stream()));
    rc = run_merged(a, limit);
  } else {
    rc = run_standard(a, limit, prec);
  }
  if (rc) return rc;
  if ((rc = store_vec(x_, a->x, a->location))) return rc;
  MFCG_CUDA(cudaEventRecord(t1, stream()));
  MFCG_CUDA(cudaMemcpyAsync(c_->h_state, c_->d_state, sizeof(SolveState), cudaMemcpyDeviceToHost, stream()));
  MFCG_CUDA(cudaStreamSynchronize(stream()));
  const SolveState& s = *c_->h_state;
  float ms = 0.f;
  MFCG_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  res->solve_ms = ms;
  if (time_kernels_) {
    double acc = 0.0;
    for (size_t i = 0; i + 1 < event_cursor_; i += 2) {
      float m = 0.f;
      MFCG_CUDA(cudaEventElapsedTime(&m, events_[i], events_[i + 1]));
      acc += m;
    }
    res->operator_ms = acc;
  }
#ifdef MFCG_TIMING
  {
    unsigned long long h[24];
    cudaMemcpyFromSymbol(h, g_phase_cycles, sizeof(h));
#if 1
    const char* names[24] = {"S.wait_lfull", "S.compute", "S.wait_tiles", "S.store", "M.wait_tiles", "M.zsweep", "M.gather", "M.barrier",
                             "P.wait_tupd", "P.wait_ldone", "P.issue", "", "U.wait_ldone", "U.wait_tfull", "U.update", "", "U.tail", "U.reduce+arrive", "S.bnd_issue", "S.bnd_wait", "S.bnd_barrier", "", "", ""};
#else
    const char* names[16] = {"P.wait_empty", "P.fill", "P.post", "", "C.wait_full", "C.x", "C.y", "C.z", "C.bar", "C.gather",
                             "", "", "", "", "", ""};
#endif
    std::fprintf(stderr, "[mfcg timing] cycles of one warp per role summed over blocks and launches (op launches %lld):\n", (long long)op_launches_);
    for (int i = 0; i < 24; ++i)
      if (names[i][0]) std::fprintf(stderr, "  %-14s %14llu\n", names[i], h[i]);
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
#endif
  res->kernel_launches = launches_;
  res->operator_launches = op_launches_;
  res->iterations = s.k;
  // solvers.py:218, 705: one operator application per iteration; launches enqueued behind the converged
  // iteration (the host polls the device state every 8 iterations in tolerance mode) return at once
  res->matvecs = s.k;
  res->residual = s.residual;
  res->breakdown = s.breakdown;
  res->breakdown_iteration = s.breakdown_iteration;
  res->breakdown_value = s.breakdown_value;
  res->converged = fixed ? (s.residual < a->tolerance) : s.converged;
  if (a->history && s.k > 0)
    MFCG_CUDA(cudaMemcpy(a->history, d_history_, sizeof(double) * 4 * (size_t)s.k, cudaMemcpyDeviceToHost));
  if (s.breakdown) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "breakdown code %d: value %.3e <= 0 at iteration %d", s.breakdown,
                  s.breakdown_value, s.breakdown_iteration);
    set_error(buf);
    return MFCG_EBREAKDOWN;
  }
  return MFCG_OK;
}

EngineBase* make_engine(OpCommon* c, int* status);  // dispatch over (degree, precision), mfcg_b200.cu

}  // namespace mfcg
