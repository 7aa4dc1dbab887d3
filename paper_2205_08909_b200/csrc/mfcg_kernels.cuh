// mfcg_kernels.cuh -- sm_100a kernels of the matrix-free CG hot path.
//
// Reference semantics (file:line relative to /root/reference/pkg/src/mfcg):
//   cell Laplacian          operator.py:253-281 + tensor.py:313-370
//   gather/scatter, BCs     operator.py:338-360
//   merged CG pre/post      solvers.py:660-698, fused_reductions solvers.py:112-127
//   scalar recurrences      solvers.py:706-764
//   standard (P)CG          solvers.py:183-340
//   Jacobi diagonal         operator.py:380-418
//
// Data layout.  The mesh is cut into bricks of
// Bx x By x Bz cells; one thread block owns one brick and marches through it
// cell layer by cell layer.  DoF vectors live in "brick numbering": the DoFs
// strictly inside a brick form one contiguous block (x fastest), all DoFs on
// brick faces/edges/corners ("shared") follow behind all interiors, entity by
// entity.  Interior DoFs are read once and written once per merged-CG
// iteration without leaving the SM; shared DoFs (about 12 % at p = 5) take the
// pre -> atomic accumulate -> post route through the small k_pre/k_post kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef MFCG_SKIP
#define MFCG_SKIP 0  // debug only: 1 skip sweeps, 2 skip gather, 4 skip post, 8 skip fill loads
#endif

// Debug build (-DMFCG_BOUNDS): index checks on every global / shared access of the brick kernel;
// a violation traps, which the host sees as a CUDA error.  (compute-sanitizer is closed on the
// GPU pool this was developed on.)
#ifdef MFCG_BOUNDS
#define MFCG_CHECK(...) do { if (!(__VA_ARGS__)) __trap(); } while (0)
#else
#define MFCG_CHECK(...)
#endif

// experiment: ring depth MFCG_STAGES for the separable kernel of degree MFCG_STAGES_P
#ifndef MFCG_STAGES
#define MFCG_STAGES 2
#define MFCG_STAGES_P 0
#endif

namespace mfcg {

typedef long long i64;

#ifdef MFCG_TIMING
// Light phase timing: one designated warp per role accumulates clock deltas in shared
// memory (single writer per slot) and flushes them once at kernel end.
static __device__ unsigned long long g_phase_cycles[24];
#define MFCG_TIC(var) long long var = clock64()
#define MFCG_TOC(var, slot)                                                                     \
  do {                                                                                          \
    if (threadIdx.x == 0 || threadIdx.x == NT_C) {                                              \
      long long now__ = clock64();                                                              \
      tcnt[slot] += (unsigned long long)(now__ - var);                                          \
      var = now__;                                                                              \
    }                                                                                           \
  } while (0)
#else
#define MFCG_TIC(var)
#define MFCG_TOC(var, slot)
#endif

struct BrickGrid {
  int p;
  int cells[3];   // cells of this rank's mesh (slab)
  int B[3];       // nominal cells per brick
  int mb[3];      // bricks per direction
  i64 n_dofs;
  i64 n_int;      // brick-interior DoFs occupy [0, n_int)
  const i64* ent_start;        // start of every macro entity, [2mbz+1][2mby+1][2mbx+1]
  const unsigned char* mask;   // per shared DoF n_int + s: bit 0 constrained, bit 1 ghost copy (owned by the lower slab)
};

// Device-resident solver state: the iteration loop never synchronises with
// the host; scalar kernels advance this struct (solvers.py:706-764).
struct SolveState {
  double am1, bm1, am2, bm2;  // alpha/beta of the two previous iterations
  double xc1, xc2;            // x catch-up coefficients for the next pre
  int xmode;                  // 0 none, 1 x += xc1 p, 2 x += xc1 p + xc2 (p - M r)
  int active;                 // 0 once converged / broken down: kernels return at once
  int k;                      // iterations completed
  int stagnant, converged, breakdown, breakdown_iteration;
  int fixed, force_x, has_prec, limit;
  double breakdown_value;
  double residual, bnorm, tol;
  double gamma, alpha, beta;  // standard (P)CG scalars
};

// Per-degree launch shape of the brick kernel: BX x BY cells per brick layer,
// NT_C "math" threads (TPC per cell) (sum-factorisation sweeps, shared memory only), NT_P
// "memory" threads (all global loads: pre on the way in, post one layer behind),
// KC points per load batch of a memory thread (memory-level parallelism).
template <int P, int G = 0> struct Cfg;
#define MFCG_CFG_X(P_, G_, BX_, BY_, TPC_, TP_, KC_, MB_, OC_)                                 \
  template <> struct Cfg<P_, G_> {                                                             \
    static constexpr int BX = BX_, BY = BY_, TPC = TPC_, NT_P = TP_, KC = KC_, MINB = MB_,     \
                         NT_C = ((BX_ * BY_ * TPC_ + 31) / 32) * 32, THREADS = NT_C + TP_;     \
    /* ONCHIP: r' and 1/diag of the layers in flight stay in shared-memory rings and the seven   \
       post sums are taken by the math warps in the gather (no re-read through L2) */            \
    static constexpr bool ONCHIP = OC_;                                                        \
  };
#define MFCG_CFG(P_, G_, BX_, BY_, TPC_, TP_, KC_, MB_) MFCG_CFG_X(P_, G_, BX_, BY_, TPC_, TP_, KC_, MB_, false)
// TPC = math threads per cell; each owns ceil((P+1)^2 / TPC) lines of that cell in every sweep.
// G = 0: separable cell operator on affine meshes (two tiles per cell);
// G = 1: general coefficient tensor per quadrature point (three tiles per cell, smaller bricks).
MFCG_CFG(1, 0, 16, 16, 1, 256, 3, 2)
MFCG_CFG(2, 0, 8, 8, 3, 256, 3, 2)
MFCG_CFG(3, 0, 8, 4, 8, 256, 3, 2)
MFCG_CFG(4, 0, 4, 4, 13, 288, 3, 2)
#ifndef MFCG_KC5
#define MFCG_KC5 3
#endif
#ifndef MFCG_TPC5
#define MFCG_TPC5 12
#endif
#ifndef MFCG_NTP5
#define MFCG_NTP5 320
#endif
#ifndef MFCG_BX5
#define MFCG_BX5 4
#define MFCG_BY5 4
#endif
#ifndef MFCG_MINB5
#define MFCG_MINB5 2
#endif
#ifndef MFCG_V7
#define MFCG_V7 0
#endif
#if MFCG_V7
#ifndef MFCG_V7_BX
#define MFCG_V7_BX 3
#define MFCG_V7_BY 3
#endif
#ifndef MFCG_V7_MINB
#define MFCG_V7_MINB 2
#endif
MFCG_CFG_X(5, 0, MFCG_V7_BX, MFCG_V7_BY, MFCG_TPC5, MFCG_NTP5, MFCG_KC5, MFCG_V7_MINB, true)
#else
MFCG_CFG_X(5, 0, MFCG_BX5, MFCG_BY5, MFCG_TPC5, MFCG_NTP5, MFCG_KC5, MFCG_MINB5, false)
#endif
MFCG_CFG(6, 0, 3, 3, 25, 256, 3, 2)
MFCG_CFG(7, 0, 2, 2, 32, 256, 3, 2)
MFCG_CFG(8, 0, 2, 2, 32, 256, 3, 2)
MFCG_CFG(1, 1, 16, 16, 1, 256, 3, 2)
MFCG_CFG(2, 1, 10, 10, 3, 192, 3, 2)
MFCG_CFG(3, 1, 6, 6, 8, 224, 3, 2)
MFCG_CFG(4, 1, 5, 5, 9, 288, 3, 2)
MFCG_CFG(5, 1, 4, 3, 18, 128, 3, 2)
MFCG_CFG(6, 1, 3, 2, 25, 224, 3, 2)
MFCG_CFG(7, 1, 2, 2, 32, 256, 3, 2)
MFCG_CFG(8, 1, 2, 2, 32, 256, 3, 2)

// G = 2: the 27-node on-the-fly variant (same shapes; separate instantiation keeps its registers
// out of the stored-geometry kernels)
MFCG_CFG(1, 2, 16, 16, 1, 96, 3, 2)
MFCG_CFG(2, 2, 10, 10, 3, 96, 3, 2)
MFCG_CFG(3, 2, 6, 6, 8, 96, 3, 2)
MFCG_CFG(4, 2, 5, 5, 9, 96, 3, 2)
MFCG_CFG(5, 2, 4, 3, 12, 96, 3, 2)
MFCG_CFG(6, 2, 3, 2, 25, 96, 3, 2)
MFCG_CFG(7, 2, 2, 2, 32, 128, 3, 2)
MFCG_CFG(8, 2, 2, 2, 32, 128, 3, 2)

// largest brick extents in x / y the kernel's shared-memory window allows (host side)
inline bool brick_caps(int p, int gclass, int* bx, int* by) {
  switch (p) {
#define MFCG_CAP(P_)                                                   \
  case P_:                                                             \
    *bx = gclass ? Cfg<P_, 1>::BX : Cfg<P_, 0>::BX;                    \
    *by = gclass ? Cfg<P_, 1>::BY : Cfg<P_, 0>::BY;                    \
    return true;
    MFCG_CAP(1) MFCG_CAP(2) MFCG_CAP(3) MFCG_CAP(4) MFCG_CAP(5) MFCG_CAP(6) MFCG_CAP(7) MFCG_CAP(8)
#undef MFCG_CAP
  }
  return false;
}

template <int P, int G = 0> struct Geo {
  static constexpr int N = P + 1;
  static constexpr int NCELL = Cfg<P, G>::BX * Cfg<P, G>::BY;
  // Math thread -> (cell, line slot) mapping.  CELL_MINOR: consecutive threads work on the SAME
  // line of consecutive cells, so the 16 lanes of a half-warp (the unit of a 64-bit shared-memory
  // access) touch one tile offset in 16 different tiles; with an odd tile stride those are 16
  // different banks in every sweep, whatever the line.  Needs a multiple of 16 cells per layer.
  static constexpr bool CELL_MINOR = (G == 0) && (NCELL % 16 == 0);
  // tile strides: element (k, j, i) of a cell tile sits at k*PSTR + j*RS + i.
  //  - CELL_MINOR: dense rows; tile stride odd and = P (P + 1 for even P) mod 16 (then the gather, whose lanes walk
  //    along x through consecutive cells, is conflict free as well)
  //  - otherwise: odd row stride (2-way conflicts in the y and z sweeps)
  static constexpr int RS = CELL_MINOR ? N : ((N % 2 == 0) ? N + 1 : N);
  static constexpr int PSTR = N * RS;
  static constexpr int tile_stride() {
    if (!CELL_MINOR) return N * PSTR;
    int t = N * PSTR;
    while (t % 2 == 0 || t % 16 != (P | 1) % 16) ++t;
    return t;
  }
  static constexpr int TILE = tile_stride();
  static constexpr int NTILE = G ? 3 : 2;               // scratch tiles per cell
  static constexpr int WX = (P * Cfg<P, G>::BX + 1) | 1; // window row stride, odd
  static constexpr int PLANE = WX * (P * Cfg<P, G>::BY + 1);
  // layers in flight between the memory and the math warps (ring depth); 2 everywhere, a build
  // parameter for experiments on the degrees whose shared memory allows more
  static constexpr int NS = (G == 0 && P == MFCG_STAGES_P) ? MFCG_STAGES : 2;
  static constexpr int RB = NS * P + 1;                 // lattice planes in the ring: consecutive layers share one
  static constexpr int NRING = Cfg<P, G>::ONCHIP ? 3 : 1;  // p' (+ r', 1/diag)
  static constexpr int HEADER = 320;                    // 27 entity starts, 3 * NS mbarriers
  template <typename T> __host__ __device__ static constexpr size_t red_offset() {
    return (HEADER + sizeof(T) * (size_t)(NRING * RB * PLANE + PLANE + NTILE * NCELL * TILE) + 15) & ~(size_t)15;
  }
  // separable path: table of the P^3 distinct 1/diag values of brick-interior DoFs (affine meshes)
  template <typename T> __host__ __device__ static constexpr size_t dtab_offset() { return red_offset<T>() + 8 * 7 * 32; }
  // separable path: per item of a layer's interior run (plane kk, row, column) the packed
  // ring offset and 1/diag class, so the memory warps decode an item with one 32-bit load
  static constexpr int ITAB_N = G == 0 ? P * (P * Cfg<P, G>::BX - 1) * (P * Cfg<P, G>::BY - 1) : 0;
  template <typename T> __host__ __device__ static constexpr size_t itab_offset() {
    return dtab_offset<T>() + (G == 0 ? ((sizeof(T) * (size_t)(P * P * P) + 15) & ~(size_t)15) : 0);
  }
  // separable path: one packed descriptor per lattice point of a layer for the gather
  static constexpr int GTAB_N = G == 0 ? (P * Cfg<P, G>::BX + 1) * (P * Cfg<P, G>::BY + 1) : 0;
  template <typename T> __host__ __device__ static constexpr size_t gtab_offset() {
    return itab_offset<T>() + ((4 * (size_t)ITAB_N + 15) & ~(size_t)15);
  }
  template <typename T> __host__ __device__ static constexpr size_t smem_bytes() {
    return gtab_offset<T>() + 8 * (size_t)GTAB_N;
  }
};

// 1D matrices of the separable (Cartesian/affine) cell operator
//   A_e = gx K (x) M (x) M + gy M (x) K (x) M + gz M (x) M (x) K,
// M = S^T W S, K = D^T W D on [0,1], g_d = det J / h_d^2.  Both matrices are
// symmetric and centro-symmetric, so a product with a line u splits into an
// even part (acting on u_j + u_{N-1-j}) and an odd part (on u_j - u_{N-1-j}),
// each a symmetric half-size matrix (the even-odd decomposition the reference
// uses in tensor.py:167-239, here additionally packed by symmetry).  For N = 6
// that is 24 distinct doubles: they fit the uniform register file, so every
// DFMA takes its coefficient as a UR operand with no shared-memory traffic.
// Passed by value (kernel parameters live in the constant bank).
template <int N> struct EOShape {
  static constexpr int H = N / 2, HE = (N + 1) / 2;
  static constexpr int NE = HE * (HE + 1) / 2, NO = H * (H + 1) / 2 > 0 ? H * (H + 1) / 2 : 1;
};
template <typename T, int N> struct SepTables {
  // K is stored once per direction, pre-scaled by g_d (saves the per-line scaling multiplies)
  T Me[EOShape<N>::NE], Mo[EOShape<N>::NO], Ke[3][EOShape<N>::NE], Ko[3][EOShape<N>::NO];
  T g[3];
  // Jacobi diagonal of the GL-collocation operator on an affine mesh, separable per direction
  // (operator.py:380-418): diag(I,J,K) = gx da[i] wa[j] wa[k] + gy wa[i] da[j] wa[k] + gz wa[i] wa[j] da[k]
  // with i = I mod p etc.; index 0 carries the sum of the two cells meeting at a cell boundary.
  // Lets the brick kernel compute 1/diag of interior DoFs instead of streaming it (8 B/DoF less).
  double wa[N], da[N];
  int diag_onfly;
};
template <typename T, int N>
__device__ __forceinline__ T diag_inverse_onfly(const SepTables<T, N>& tab, int i, int j, int k) {
  const double wi = tab.wa[i], wj = tab.wa[j], wk = tab.wa[k];
  const double d = (double)tab.g[0] * tab.da[i] * wj * wk + (double)tab.g[1] * wi * tab.da[j] * wk +
                   (double)tab.g[2] * wi * wj * tab.da[k];
  return (T)(1.0 / d);
}
__host__ __device__ constexpr int sym_idx(int i, int j) { return i <= j ? j * (j + 1) / 2 + i : i * (i + 1) / 2 + j; }

// e_j = u_j + u_{N-1-j}, o_j = u_j - u_{N-1-j}; the middle entry (odd N) goes to e
template <int N, typename T>
__device__ __forceinline__ void eo_split(const T* u, T* e, T* o) {
  constexpr int H = EOShape<N>::H;
#pragma unroll
  for (int j = 0; j < H; ++j) { e[j] = u[j] + u[N - 1 - j]; o[j] = u[j] - u[N - 1 - j]; }
  if (N & 1) e[H] = u[H];
}
// se += Ae e, so += Ao o with packed symmetric halves
template <int N, typename T>
__device__ __forceinline__ void eo_mul(const T* Ae, const T* Ao, const T* e, const T* o, T* se, T* so) {
  constexpr int H = EOShape<N>::H, HE = EOShape<N>::HE;
#pragma unroll
  for (int i = 0; i < HE; ++i)
#pragma unroll
    for (int j = 0; j < HE; ++j) se[i] += Ae[sym_idx(i, j)] * e[j];
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int j = 0; j < H; ++j) so[i] += Ao[sym_idx(i, j)] * o[j];
}
// out_i = se_i + so_i, out_{N-1-i} = se_i - so_i
template <int N, typename T>
__device__ __forceinline__ void eo_join(const T* se, const T* so, T* out) {
  constexpr int H = EOShape<N>::H;
#pragma unroll
  for (int i = 0; i < H; ++i) { out[i] = se[i] + so[i]; out[N - 1 - i] = se[i] - so[i]; }
  if (N & 1) out[H] = se[H];
}

__device__ __forceinline__ int brick_cells(const BrickGrid& g, int d, int m) {
  int r = g.cells[d] - m * g.B[d];
  return r < g.B[d] ? r : g.B[d];
}

__device__ __forceinline__ void warp_reduce7(double* s) {
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
}

// Block-level reduction of seven sums; result row written by thread 0.
// red: >= 7*32 doubles of shared memory.
__device__ __forceinline__ void block_reduce7_store(double* s, double* red, double* out_row) {
  warp_reduce7(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 7; ++q) red[w * 7 + q] = s[q];
  __syncthreads();
  if (threadIdx.x < 7) {
    double acc = 0.0;
    for (int i = 0; i < nw; ++i) acc += red[i * 7 + threadIdx.x];
    out_row[threadIdx.x] = acc;
  }
}

// ---------------------------------------------------------------------------
// General geometry (curved meshes): per quadrature point the symmetric coefficient tensor
// G = J^-1 (w det J) J^-T (operator.py:202-249, mesh.py:194-201 storage xx,yy,zz,xy,xz,yz).
// The cell kernel interpolates to the n_q = p+1 quadrature points (S, centro-symmetric),
// differentiates there with the collocation derivative Dc (anti-centro-symmetric; Dc S = D up
// to rounding, tensor.py: the 9+9 sweeps of evaluate/integrate_gradients collapse to 12),
// applies G, and transposes.  Even/odd halves, row-major, not symmetric:
//   Se[q][i] = (S[q][i] + S[q][N-1-i])/2 (middle column S[q][H]),  So[q][i] = (S[q][i] - S[q][N-1-i])/2,
//   Be[q][r] = (Dc[q][r] + Dc[q][N-1-r])/2 (middle column Dc[q][H]), Bo[q][r] = (Dc[q][r] - Dc[q][N-1-r])/2.
template <typename T, int N> struct GenTables {
  static constexpr int H = N / 2, HE = (N + 1) / 2;
  T Se[HE * HE], So[(H > 0 ? H : 1) * (H > 0 ? H : 1)], Be[(H > 0 ? H : 1) * HE], Bo[HE * (H > 0 ? H : 1)];
  T qv[N * 3], qd[N * 3];  // quadratic Lagrange basis on {0,1/2,1} and its derivative at the quadrature points
  T w3[N];                 // quadrature weights (quadratic_compute builds w_q det J itself)
};
struct GeomAccess {
  int kind;              // MFCG_GEOM_*: 1 final tensor, 2 inverse Jacobian + jxw, 3 27 nodes per cell
  const void* data;      // [n_cells][nq^3][6] | [n_cells][nq^3][9] | [n_cells][27][3]
  const void* jxw;       // kind 2: [n_cells][nq^3]
};

// out = A u for centro-symmetric A given by halves (transposed = apply A^T)
template <int N, typename T>
__device__ __forceinline__ void eo_apply_sym(const T* Ae, const T* Ao, bool transposed, const T* e, const T* o, T* se, T* so) {
  constexpr int H = EOShape<N>::H, HE = EOShape<N>::HE;
#pragma unroll
  for (int i = 0; i < HE; ++i) {
    T a = 0;
#pragma unroll
    for (int j = 0; j < HE; ++j) a += (transposed ? Ae[j * HE + i] : Ae[i * HE + j]) * e[j];
    se[i] = a;
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T a = 0;
#pragma unroll
    for (int j = 0; j < H; ++j) a += (transposed ? Ao[j * H + i] : Ao[i * H + j]) * o[j];
    so[i] = a;
  }
}
// out = Dc u (or Dc^T u) for anti-centro-symmetric Dc: even output from odd input and vice versa.
// Be is H x HE (rows q < H), Bo is HE x H (rows q < HE).
template <int N, typename T>
__device__ __forceinline__ void eo_apply_anti(const T* Be, const T* Bo, bool transposed, const T* e, const T* o, T* se, T* so) {
  constexpr int H = EOShape<N>::H, HE = EOShape<N>::HE;
#pragma unroll
  for (int i = 0; i < HE; ++i) {  // even part of the output
    T a = 0;
#pragma unroll
    for (int j = 0; j < H; ++j) a += (transposed ? Be[j * HE + i] : Bo[i * H + j]) * o[j];
    se[i] = a;
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {   // odd part of the output
    T a = 0;
#pragma unroll
    for (int j = 0; j < HE; ++j) a += (transposed ? Bo[j * H + i] : Be[i * HE + j]) * e[j];
    so[i] = a;
  }
}

// Jacobian of the tri-quadratic cell map at one point from the 27 nodes (x fastest),
// J[i][j] = d x_i / d xi_j (mesh.py:155-174), given the 1D quadratic basis values/derivatives
// (3 each) in every direction.
__device__ __forceinline__ void jacobian27(const double* nodes, const double* vx, const double* dx, const double* vy,
                                           const double* dy, const double* vz, const double* dz, double* J) {
#pragma unroll
  for (int t = 0; t < 9; ++t) J[t] = 0.0;
  for (int c = 0; c < 3; ++c)
    for (int b = 0; b < 3; ++b) {
      const double vv = vy[b] * vz[c], dyv = dy[b] * vz[c], dzv = vy[b] * dz[c];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double* nd = nodes + 3 * ((c * 3 + b) * 3 + a);
        const double wx = dx[a] * vv, wy = vx[a] * dyv, wz = vx[a] * dzv;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          J[i * 3 + 0] += nd[i] * wx;
          J[i * 3 + 1] += nd[i] * wy;
          J[i * 3 + 2] += nd[i] * wz;
        }
      }
    }
}
// inverse and determinant of a 3x3 matrix
__device__ __forceinline__ double invert3(const double* J, double* inv) {
  const double c00 = J[4] * J[8] - J[5] * J[7], c01 = J[5] * J[6] - J[3] * J[8], c02 = J[3] * J[7] - J[4] * J[6];
  const double det = J[0] * c00 + J[1] * c01 + J[2] * c02;
  const double id = 1.0 / det;
  inv[0] = c00 * id; inv[1] = (J[2] * J[7] - J[1] * J[8]) * id; inv[2] = (J[1] * J[5] - J[2] * J[4]) * id;
  inv[3] = c01 * id; inv[4] = (J[0] * J[8] - J[2] * J[6]) * id; inv[5] = (J[2] * J[3] - J[0] * J[5]) * id;
  inv[6] = c02 * id; inv[7] = (J[1] * J[6] - J[0] * J[7]) * id; inv[8] = (J[0] * J[4] - J[1] * J[3]) * id;
  return det;
}
// G = inv (jxw) inv^T, 6-storage
__device__ __forceinline__ void tensor6(const double* inv, double jxw, double* g) {
  g[0] = jxw * (inv[0] * inv[0] + inv[1] * inv[1] + inv[2] * inv[2]);
  g[1] = jxw * (inv[3] * inv[3] + inv[4] * inv[4] + inv[5] * inv[5]);
  g[2] = jxw * (inv[6] * inv[6] + inv[7] * inv[7] + inv[8] * inv[8]);
  g[3] = jxw * (inv[0] * inv[3] + inv[1] * inv[4] + inv[2] * inv[5]);
  g[4] = jxw * (inv[0] * inv[6] + inv[1] * inv[7] + inv[2] * inv[8]);
  g[5] = jxw * (inv[3] * inv[6] + inv[4] * inv[7] + inv[5] * inv[8]);
}

// ---------------------------------------------------------------------------
// Line order of the sweeps.  A math thread q of a cell handles lines order(t*TPC+q),
// t = 0,1,...; -1 = idle lane.  The order decides which shared-memory banks the 16 lanes of a
// half-warp (the unit of a 64-bit access) hit.
template <int N> struct LineOrder {
  static constexpr bool custom = false;
  __device__ static __forceinline__ int x(int s, int tpc) { return s < N * N ? s : -1; }
  __device__ static __forceinline__ int y(int s, int tpc) { return s < N * N ? s : -1; }
  __device__ static __forceinline__ int z(int s, int tpc) { return s < N * N ? s : -1; }
};
#ifdef MFCG_LINE_ORDER
// Experiment: line orders found by exhaustive search for the padded-row layout (RS = 7, plane 42,
// tile 252 = 12 mod 16) and 12 threads per cell: every half-warp (12 + 4, 8 + 8, 4 + 12 lanes of
// two cells) hits 16 different banks in the x stores and the y sweep; z stays 2-way.
template <> struct LineOrder<6> {
  static constexpr bool custom = true;
  __device__ static __forceinline__ int x(int s, int tpc) {
    if (tpc != 12) return s < 36 ? s : -1;
    constexpr signed char t[36] = {24, 35, 26, 33, 20, 31, 22, 29, 32, 27, 34, 25, 4, 11, 6, 9, 16, 23,
                                   18, 21, 28, 19, 30, 17, 0, 7, 2, 5, 12, 3, 14, 1, 8, 15, 10, 13};
    return t[s];
  }
  __device__ static __forceinline__ int y(int s, int tpc) {
    if (tpc != 12) return s < 36 ? s : -1;
    constexpr signed char t[36] = {32, 33, 26, 27, 24, 25, 18, 19, 28, 29, 30, 31, 8, 9, 10, 11, 20, 21,
                                   22, 23, 12, 13, 34, 35, 0, 1, 2, 3, 4, 5, 14, 15, 16, 17, 6, 7};
    return t[s];
  }
  __device__ static __forceinline__ int z(int s, int tpc) { return s < 36 ? s : -1; }
};
#endif

// ---------------------------------------------------------------------------
// mbarrier / named-barrier helpers (shared::cta)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef MFCG_WAIT_HINT
#define MFCG_WAIT_HINT 20000
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
#ifdef MFCG_WAIT_SLEEP
  for (;;) {  // explicit back-off between polls
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    if (ok) break;
    __nanosleep(MFCG_WAIT_SLEEP);
  }
#else
  do {  // the hint lets the hardware park the warp until the phase flips instead of spinning
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"((unsigned)MFCG_WAIT_HINT)
        : "memory");
  } while (!ok);
#endif
}
// L2 prefetch of a contiguous run (TMA-class bulk prefetch, no registers or shared memory):
// [ptr + first, ptr + first + count) elements, widened to 16-byte alignment inside [0, limit)
template <typename T>
__device__ __forceinline__ void prefetch_l2_run(const T* ptr, i64 first, i64 count, i64 limit) {
  if (count <= 0) return;
  constexpr i64 PER16 = 16 / sizeof(T);
  i64 lo = first - (first % PER16);
  i64 hi = first + count;
  hi += (PER16 - hi % PER16) % PER16;
  if (hi > limit) hi -= PER16;
  if (hi <= lo) return;
  const unsigned bytes = (unsigned)((hi - lo) * (i64)sizeof(T));
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr + lo), "r"(bytes) : "memory");
}

// -DMFCG_LEADER_POLL: one warp of a role polls the mbarrier, the role's other warps sleep in a
// hardware named barrier.  Polling by every warp is 37 % of all issued instructions, yet the
// leader variant measured 1.5 % slower (profiles/r01_notes.md), so every warp polls by default.
template <int COUNT> __device__ __forceinline__ void role_wait(unsigned long long* bar, unsigned parity, bool leader, int id) {
#ifndef MFCG_LEADER_POLL
  mbar_wait(bar, parity);
#else
  if (leader) mbar_wait(bar, parity);
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(COUNT) : "memory");
#endif
}
#ifndef MFCG_UNROLL_T
#define MFCG_UNROLL_T 1
#endif
// how the memory warps load the interior runs: 0 plain, 1 ld.global.cg (L2 only), 2 ld.global.cs (streaming)
#ifndef MFCG_LOAD_HINT
#define MFCG_LOAD_HINT 0
#endif
#if MFCG_LOAD_HINT == 1
#define MFCG_LDG(p) __ldcg(p)
#elif MFCG_LOAD_HINT == 2
#define MFCG_LDG(p) __ldcs(p)
#else
#define MFCG_LDG(p) (*(p))
#endif
#ifndef MFCG_GEO_PREFETCH
#define MFCG_GEO_PREFETCH 0  // bulk L2 prefetch of the next layer's stored geometry (curved meshes)
#endif
template <int COUNT> __device__ __forceinline__ void math_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(COUNT) : "memory");
}

// ---------------------------------------------------------------------------
// The brick kernel.  MODE 0: dst = A src (operator.py:285-360).
// MODE 1: one merged-CG iteration on brick-interior DoFs (solvers.py:660-704).
//
// One block = one brick, marched layer by layer in z.  Warp-specialised:
//   memory warps  stream the next layer's lattice planes from HBM (MODE 1: r, v,
//                 p, 1/diag, x of every interior DoF -> pre update -> r, p, x
//                 written back, p into the shared-memory plane ring) while the
//                 math warps work on the current layer, and run the seven post
//                 sums one layer behind on values still resident in L2;
//   math warps    never load from global memory: x/y/z even-odd sweeps in shared
//                 memory, a deterministic gather of the cells' contributions per
//                 lattice point, v stored (interior) or atomically added (shared).
// Hand-over through two mbarrier pairs (full/empty per layer parity).
template <int P, typename T, int MODE, int G, bool MC = false>
__global__ void __launch_bounds__(Cfg<P, G>::THREADS, Cfg<P, G>::MINB)
k_brick(BrickGrid g, SepTables<T, P + 1> tab, GenTables<T, P + 1> gen, GeomAccess geo,
        const T* __restrict__ src, T* __restrict__ Pv,
        T* __restrict__ V, T* __restrict__ R, T* __restrict__ X, const T* __restrict__ Minv,
        const SolveState* __restrict__ st, double* __restrict__ partials, int brick_offset,
        int ncomp = 1, i64 comp_stride = 0, i64 part_stride = 0) {
  constexpr int N = P + 1, RS = Geo<P, G>::RS, PSTR = Geo<P, G>::PSTR, TILE = Geo<P, G>::TILE, WX = Geo<P, G>::WX,
                PLANE = Geo<P, G>::PLANE, NCELL = Geo<P, G>::NCELL, RB = Geo<P, G>::RB,
                NT_C = Cfg<P, G>::NT_C, NT_P = Cfg<P, G>::NT_P, KC = Cfg<P, G>::KC, HE = EOShape<N>::HE,
                NS = Geo<P, G>::NS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  i64* st27 = reinterpret_cast<i64*>(smem_raw);                               // 27 entity starts
  // full[2] (memory -> math), ringfree[2] (ring planes of a layer read), vdone[2] (v of a layer stored)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw + 224);
  constexpr bool ONCHIP = Cfg<P, G>::ONCHIP && MODE == 1;
  T* ring = reinterpret_cast<T*>(smem_raw + Geo<P, G>::HEADER);
  T* Rring = ring + RB * PLANE;              // only with Cfg::ONCHIP
  T* Mring = Rring + RB * PLANE;
  T* carry = ring + Geo<P, G>::NRING * RB * PLANE;
  T* A = carry + PLANE;
  T* Bs = A + NCELL * TILE;
  constexpr size_t RED_OFF = Geo<P, G>::template red_offset<T>();
  double* red = reinterpret_cast<double*>(smem_raw + RED_OFF);
  T* dtab = reinterpret_cast<T*>(smem_raw + Geo<P, G>::template dtab_offset<T>());
  unsigned* itab = reinterpret_cast<unsigned*>(smem_raw + Geo<P, G>::template itab_offset<T>());
  constexpr bool USE_ITAB = G == 0;
  uint2* gtab = reinterpret_cast<uint2*>(smem_raw + Geo<P, G>::template gtab_offset<T>());
  constexpr bool USE_GTAB = G == 0;
  static_assert(!USE_ITAB || (PLANE < 1024 && P * P * P <= 512 && P < 8 + 1), "packed item table fields");

#ifdef MFCG_TIMING
  __shared__ unsigned long long tcnt[16];
  if (threadIdx.x < 16) tcnt[threadIdx.x] = 0;
#endif
  const int tid = threadIdx.x;
  T am1 = 0, bm1 = 0, xc1 = 0, xc2 = 0;
  int xmode = 0;
  if (MODE == 1) {
    if (!st->active) return;
    am1 = (T)st->am1; bm1 = (T)st->bm1; xc1 = (T)st->xc1; xc2 = (T)st->xc2; xmode = st->xmode;
  }

  // ncomp > 1 (stored geometry, several components in one launch): consecutive blocks work on the same brick, one
  // component each, so the brick's geometry block comes from HBM once and from L2 for the other components
  // (a separate instantiation, MC: adjusting the pointer arguments costs the single-component kernels registers)
  int bidx = blockIdx.x;
  if constexpr (MC) {
    const int comp = bidx % ncomp;
    bidx /= ncomp;
    const i64 o = comp * comp_stride;
    if (src) src += o;
    if (Pv) Pv += o;
    V += o;
    if (R) R += o;
    if (X) X += o;
    if (Minv) Minv += o;
    if (partials) partials += comp * part_stride;
  }
  int b = bidx + brick_offset;  // slab runs launch the interface brick layers first; a range may wrap around
  if (b >= g.mb[0] * g.mb[1] * g.mb[2]) b -= g.mb[0] * g.mb[1] * g.mb[2];
  const int mx = b % g.mb[0];
  const int my = (b / g.mb[0]) % g.mb[1];
  const int mz = b / (g.mb[0] * g.mb[1]);
  const int bcx = brick_cells(g, 0, mx), bcy = brick_cells(g, 1, my), bcz = brick_cells(g, 2, mz);
  const int Lx = P * bcx, Ly = P * bcy, Lz = P * bcz;
  if (tid < 27) {
    const int ex = tid % 3, ey = (tid / 3) % 3, ez = tid / 9;
    st27[tid] = g.ent_start[((i64)(2 * mz + ez) * (2 * g.mb[1] + 1) + (2 * my + ey)) * (2 * g.mb[0] + 1) + 2 * mx + ex];
  }
  if (tid == 32) {
    for (int sidx = 0; sidx < NS; ++sidx) {
      mbar_init(&bars[sidx], NT_P);            // full
      mbar_init(&bars[NS + sidx], NT_C);       // ring free
      mbar_init(&bars[2 * NS + sidx], NT_C);   // v stored
    }
  }
  for (int i = tid; i < PLANE; i += NT_C + NT_P) carry[i] = (T)0;
  if (MODE == 1 && G == 0 && tab.diag_onfly)
    for (int i = tid; i < P * P * P; i += NT_C + NT_P)
      dtab[i] = diag_inverse_onfly<T, N>(tab, i % P, (i / P) % P, i / (P * P));
  // Gather descriptor of lattice point rem = j * (Lx+1) + i of a layer (independent of the layer):
  //  x: tile offset of the point in cell (i/P, j/P) [14 bits], which of the four cells around it
  //     exist (bits 14-17: (cx,cy), (cx-1,cy), (cx,cy-1), (cx-1,cy-1)), brick-boundary flag, entity
  //  y: offset in the lattice plane, offset inside the macro entity, plane-stride selector
  auto gather_descriptor = [&](int rem) -> uint2 {
    const int fw_ = Lx + 1;
    const int j = rem / fw_, i = rem - j * fw_;
    const int ex = i == 0 ? 0 : (i == Lx ? 2 : 1), ey = j == 0 ? 0 : (j == Ly ? 2 : 1);
    const int ox = ex == 1 ? i - 1 : 0, oy = ey == 1 ? j - 1 : 0;
    const int lx = ex == 1 ? Lx - 1 : 1;
    const int cx1 = i / P, ix1 = i - cx1 * P, cy1 = j / P, iy1 = j - cy1 * P;
    const unsigned base = (unsigned)((cy1 * bcx + cx1) * TILE + iy1 * RS + ix1);
    const unsigned v11 = cx1 < bcx && cy1 < bcy, v10 = ix1 == 0 && cx1 > 0 && cy1 < bcy,
                   v01 = iy1 == 0 && cy1 > 0 && cx1 < bcx, v00 = ix1 == 0 && iy1 == 0 && cx1 > 0 && cy1 > 0;
    const unsigned edge = (ex != 1) || (ey != 1);
    const unsigned sel = (ex == 1 ? 1u : 0u) | (ey == 1 ? 2u : 0u);
    uint2 d;
    d.x = base | (v11 << 14) | (v10 << 15) | (v01 << 16) | (v00 << 17) | (edge << 18) | ((unsigned)(ex + 3 * ey) << 19);
    d.y = (unsigned)(j * WX + i) | ((unsigned)(ox + lx * oy) << 10) | (sel << 22);
    return d;
  };
  if (USE_GTAB) {
    // table order: first the points strictly inside a cell in x and y (one contribution, plain
    // stores: warps of the gather stay uniform), then the brick-boundary points in the perimeter
    // order of the memory warps (which read the same descriptors), then the other cell-boundary points
    const int fw_ = Lx + 1, rowc = bcx * (P - 1), n_in = rowc * bcy * (P - 1);
    const int nper = 2 * fw_ + 2 * (Ly - 1);
    for (int rem = tid; rem < fw_ * (Ly + 1); rem += NT_C + NT_P) {
      const int j = rem / fw_, i = rem - j * fw_;
      const int cx1 = i / P, ix1 = i - cx1 * P, cy1 = j / P, iy1 = j - cy1 * P;
      const int rows_before = cy1 * (P - 1) + (iy1 == 0 ? 0 : iy1 - 1);
      const int in_row_before = cx1 * (P - 1) + (ix1 == 0 ? 0 : ix1 - 1);
      const int before = rows_before * rowc + (iy1 != 0 ? in_row_before : 0);  // inner points with smaller rem
      int pos;
      if (ix1 != 0 && iy1 != 0) pos = before;
      else if (j == 0) pos = n_in + i;
      else if (j == Ly) pos = n_in + fw_ + i;
      else if (i == 0 || i == Lx) pos = n_in + 2 * fw_ + 2 * (j - 1) + (i == Lx ? 1 : 0);
      else pos = n_in + nper + (rem - before - (fw_ + 2 * (j - 1) + 1));
      MFCG_CHECK(pos >= 0 && pos < Geo<P, G>::GTAB_N);
      gtab[pos] = gather_descriptor(rem);
    }
  }
  if (USE_ITAB) {
    // item it = (kk * (Ly-1) + jm) * (Lx-1) + im of a layer's interior run: lattice plane Kfirst + kk
    // with Kfirst = 1 (mod P), row jm + 1, column im + 1
    const int lxm_ = Lx - 1, n2d_ = (Lx - 1) * (Ly - 1);
    for (int it = tid; it < P * n2d_; it += NT_C + NT_P) {
      const int kk = it / n2d_, rem2 = it - kk * n2d_, jm = rem2 / lxm_, im = rem2 - jm * lxm_;
      const unsigned inplane = (unsigned)((jm + 1) * WX + im + 1);
      const unsigned didx = (unsigned)((((1 + kk) % P) * P + (jm + 1) % P) * P + (im + 1) % P);
      MFCG_CHECK(it < Geo<P, G>::ITAB_N && inplane < 1024u && didx < (unsigned)(P * P * P));
      itab[it] = (unsigned)kk | (inplane << 4) | (didx << 14);
    }
  }
  __syncthreads();

  const int fw = Lx + 1, fp = fw * (Ly + 1);
  const int nint2d_c = (Lx - 1) * (Ly - 1);  // interior points of one lattice plane
  const int n_in_c = bcx * (P - 1) * bcy * (P - 1);  // lattice points of a plane strictly inside a cell
  const i64 n_int = g.n_int;

  if (tid >= NT_C) {
    // ===================== memory warps =====================
    const int ptid = tid - NT_C;
    const int pwarp = ptid >> 5;
    const int nint2d = (Lx - 1) * (Ly - 1);                  // interior points of one lattice plane
    const int nperim = fp - nint2d;                           // brick-boundary points of one plane
    const int lxm = Lx > 1 ? Lx - 1 : 1;
    const unsigned lxm_magic = (65536u + lxm - 1) / lxm;
    const unsigned n2d_magic = nint2d > 0 ? (unsigned)((0x100000000ull + nint2d - 1) / nint2d) : 0u;
    const unsigned per_magic = (unsigned)((0x100000000ull + nperim - 1) / nperim);
    const i64 st_int = st27[13];
    // interior run of layer Lq in every vector: [run_first(Lq), +run_count(Lq))
    auto prefetch_layer = [&](int Lq) {
#if MFCG_GEO_PREFETCH
      // stored geometry of the layer's cells (one contiguous block per cell), read by the math warps
      if (G == 1 && Lq < bcz && ptid >= 32 && ptid < 32 + bcx * bcy) {
        const int c = ptid - 32, cy = c / bcx, cx = c - cy * bcx;
        const i64 cellg = ((i64)(mz * g.B[2] + Lq) * g.cells[1] + (my * g.B[1] + cy)) * g.cells[0] + (mx * g.B[0] + cx);
        constexpr int NQ3 = N * N * N;
        const unsigned per = geo.kind == 1 ? 6u : 9u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const T*>(geo.data) + cellg * NQ3 * per),
                     "r"((unsigned)(NQ3 * per * sizeof(T))) : "memory");
        if (geo.kind == 2)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const T*>(geo.jxw) + cellg * NQ3),
                       "r"((unsigned)(NQ3 * sizeof(T))) : "memory");
      }
#endif
      if (Lq >= bcz || nint2d <= 0 || ptid >= 5) return;
      const int kq0 = Lq == 0 ? 0 : 1;
      const int Kf = Lq * P + kq0 > 1 ? Lq * P + kq0 : 1;
      const int Kl = Lq * P + P < Lz - 1 ? Lq * P + P : Lz - 1;
      if (Kl < Kf) return;
      const i64 first = st_int + (i64)nint2d * (Kf - 1), count = (i64)(Kl - Kf + 1) * nint2d;
      if (MODE == 0) {
        if (ptid == 0) prefetch_l2_run(src, first, count, g.n_dofs);
      } else {
        if (ptid == 0) prefetch_l2_run(Pv, first, count, g.n_dofs);
        if (ptid == 1) prefetch_l2_run(R, first, count, g.n_dofs);
        if (ptid == 2) prefetch_l2_run(V, first, count, g.n_dofs);
        if (ptid == 3 && !(G == 0 && tab.diag_onfly)) prefetch_l2_run(Minv, first, count, g.n_dofs);
        if (ptid == 4 && xmode) prefetch_l2_run(X, first, count, g.n_dofs);
      }
    };
    // L2 prefetch distance in layers (TMA-class bulk prefetch of the next layer's interior runs).
    // Measured (profiles/r01_notes.md): one layer ahead shortens the kernel by 6 % once the sweeps
    // are bank-conflict free (the memory warps then wait on load latency), DRAM traffic +2 %;
    // two layers ahead is worse than one.
#ifndef MFCG_L2_PREFETCH
#define MFCG_L2_PREFETCH 1
#endif
    constexpr int PF = MFCG_L2_PREFETCH;
    for (int Lq = 0; Lq < PF; ++Lq) prefetch_layer(Lq);
    // separable path: the thread's share of the seven sums stays in registers over the whole brick;
    // the curved paths (register-bound math warps) reduce per layer into the shared-memory slots
    constexpr bool PER_BRICK_SUMS = G == 0;
    double s[7] = {0, 0, 0, 0, 0, 0, 0};
    if (!PER_BRICK_SUMS && !ONCHIP && (ptid & 31) == 0)
      for (int q = 0; q < 7; ++q) red[pwarp * 7 + q] = 0.0;
    MFCG_TIC(tp);
    for (int L = 0; L < bcz + NS; ++L) {  // the post of a layer runs NS iterations after its fill
      const int stage = L % NS;
      if (PF > 0) prefetch_layer(L + PF);
      // post sums of layer L - NS.  Separable path: before the fill of layer L (its loads were
      // prefetched to L2 at the top of the iteration and get the time of the post to arrive, -2 %);
      // curved paths: after it (measured 1.5 % better there)
      constexpr bool POST_FIRST = G == 0;
      auto do_post = [&]() {
      if (MODE == 1 && !ONCHIP && L >= NS && !(MFCG_SKIP & 4)) {
        role_wait<NT_P>(&bars[2 * NS + stage], ((L / NS) - 1) & 1, pwarp == 0, 2);  // v of layer L-NS stored
        // ---- post sums of layer L-2 (solvers.py:692-698): its v is final and, like r, p and
        // 1/diag, still resident in L2; one contiguous run per vector
        const int Lp = L - NS;
        const int Klo = Lp == 0 ? 1 : Lp * P, Khi = Lp * P + P - 1;
        const int nitem = nint2d > 0 ? (Khi - Klo + 1) * nint2d : 0;
        const i64 gbase = st_int + (i64)nint2d * (Klo - 1);
        for (int it0 = ptid; it0 < nitem; it0 += KC * NT_P) {
          T rr[KC], vv[KC], pp[KC], mm[KC];
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const int it = it0 + c * NT_P;
            rr[c] = vv[c] = pp[c] = mm[c] = (T)0;
            if (it < nitem) {
              const i64 gi = gbase + it;
              MFCG_CHECK(gi >= 0 && gi < n_int);
              rr[c] = MFCG_LDG(R + gi); vv[c] = MFCG_LDG(V + gi); pp[c] = MFCG_LDG(Pv + gi);
              if (G == 0 && tab.diag_onfly) {
                // plane Klo + kk: the table is laid out for planes = 1 + kk (mod P)
                const int itp = Lp == 0 ? it : (it >= nint2d ? it - nint2d : it + (P - 1) * nint2d);
                MFCG_CHECK(itp >= 0 && itp < Geo<P, G>::ITAB_N && (itab[itp] >> 14) < (unsigned)(P * P * P));
                mm[c] = dtab[itab[itp] >> 14];
              } else {
                mm[c] = Minv[gi];
              }
            }
          }
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const double r = (double)rr[c], m = (double)mm[c], p = (double)pp[c], v = (double)vv[c];
            const double mr = m * r, mv = m * v;
            s[0] += r * r; s[1] += p * v; s[2] += r * v; s[3] += v * v;
            s[4] += r * mr; s[5] += r * mv; s[6] += v * mv;
          }
        }
        if (!PER_BRICK_SUMS) {
          warp_reduce7(s);
          if ((ptid & 31) == 0)
#pragma unroll
            for (int q = 0; q < 7; ++q) red[pwarp * 7 + q] += s[q];
#pragma unroll
          for (int q = 0; q < 7; ++q) s[q] = 0.0;
        }
        MFCG_TOC(tp, 2);
      }
      };
      if (POST_FIRST) do_post();
      // the ring planes layer L overwrites were last read by the x sweep of layer L-NS
      if (L >= NS && L < bcz) role_wait<NT_P>(&bars[NS + stage], ((L / NS) - 1) & 1, pwarp == 0, 2);
      MFCG_TOC(tp, 0);
      if (L < bcz) {
        // ---- fill the ring with the planes layer L adds (plane 0 is shared with layer L-1)
        const int k0 = L == 0 ? 0 : 1;
        // (a) brick-interior points: one contiguous run per vector, pre fused (solvers.py:660-690)
        const int Kfirst = L * P + k0 > 1 ? L * P + k0 : 1;
        const int Klast = L * P + P < Lz - 1 ? L * P + P : Lz - 1;
        const int nitem = (nint2d > 0 && Klast >= Kfirst && !(MFCG_SKIP & 8)) ? (Klast - Kfirst + 1) * nint2d : 0;
        const i64 gbase = st_int + (i64)nint2d * (Kfirst - 1);
        const int kslot = Kfirst % RB;
        for (int it0 = ptid; it0 < nitem; it0 += KC * NT_P) {
          T rr[KC], vv[KC], pp[KC], mm[KC], xx[KC];
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const int it = it0 + c * NT_P;
            rr[c] = vv[c] = pp[c] = mm[c] = xx[c] = (T)0;
            if (it < nitem) {
              const i64 gi = gbase + it;
              MFCG_CHECK(gi >= 0 && gi < n_int);
              if (MODE == 0) {
                pp[c] = src[gi];
              } else {
                pp[c] = MFCG_LDG(Pv + gi); rr[c] = MFCG_LDG(R + gi); vv[c] = MFCG_LDG(V + gi);
                if (!tab.diag_onfly) mm[c] = MFCG_LDG(Minv + gi);
                if (xmode) xx[c] = MFCG_LDG(X + gi);
              }
            }
          }
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const int it = it0 + c * NT_P;
            if (it >= nitem) continue;
            int kk, inplane, didx = 0;
            if (USE_ITAB) {
              MFCG_CHECK(it >= 0 && it < Geo<P, G>::ITAB_N);
              const unsigned e = itab[it];
              kk = (int)(e & 15u); inplane = (int)((e >> 4) & 1023u); didx = (int)(e >> 14);
            } else {
              kk = (int)__umulhi((unsigned)it, n2d_magic);
              const int rem2 = it - kk * nint2d;
              const int jm = (int)(((unsigned)rem2 * lxm_magic) >> 16);
              const int im = rem2 - jm * lxm;
              inplane = (jm + 1) * WX + im + 1;
            }
            MFCG_CHECK(kk >= 0 && Kfirst + kk <= Klast && inplane > WX && inplane < PLANE);
            T val = pp[c];
            T rnew = (T)0;
            if (MODE == 1) {
              const i64 gi = gbase + it;
              if (G == 0 && tab.diag_onfly) mm[c] = dtab[didx];
              T r = rr[c], p = pp[c];
              if (xmode) {
                T x = xx[c];
                if (xmode == 2) x += xc1 * p + xc2 * (p - mm[c] * r);
                else x += xc1 * p;
                X[gi] = x;
              }
              r -= am1 * vv[c];
              p = mm[c] * r + bm1 * p;
              R[gi] = r;
              Pv[gi] = p;
              val = p;
              rnew = r;
            }
            int slot = kslot + kk;
            if (slot >= RB) slot -= RB;
            const int rdst = slot * PLANE + inplane;
            ring[rdst] = val;
            if (ONCHIP) { Rring[rdst] = rnew; Mring[rdst] = mm[c]; }
          }
        }
        // (b) brick-boundary points of the layer's planes: already pre-updated by k_pre; p only
        {
          const int nk = P + 1 - k0;
          const int nsh = nk * nperim;
          for (int it0 = ptid; it0 < nsh; it0 += 2 * NT_P) {
            T pp[2];
            unsigned char mk[2];
            int dst[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int it = it0 + c * NT_P;
              pp[c] = (T)0; mk[c] = 0; dst[c] = -1;
              if (it < nsh) {
                const int kk = (int)__umulhi((unsigned)it, per_magic);
                const int e = it - kk * nperim;
                int e2, o2, cw, pstride;
                if (USE_GTAB) {
                  MFCG_CHECK(e >= 0 && n_in_c + e < Geo<P, G>::GTAB_N);
                  const uint2 d = gtab[n_in_c + e];
                  e2 = (int)((d.x >> 19) & 15u); cw = (int)(d.y & 1023u); o2 = (int)((d.y >> 10) & 4095u);
                  const unsigned sel = d.y >> 22;
                  pstride = ((sel & 1u) ? Lx - 1 : 1) * ((sel & 2u) ? Ly - 1 : 1);
                } else {
                  int i, j;
                  if (e < fw) { j = 0; i = e; }
                  else if (e < 2 * fw) { j = Ly; i = e - fw; }
                  else { const int r2 = e - 2 * fw; j = 1 + (r2 >> 1); i = (r2 & 1) ? Lx : 0; }
                  const int ex = i == 0 ? 0 : (i == Lx ? 2 : 1), ey = j == 0 ? 0 : (j == Ly ? 2 : 1);
                  const int ox = ex == 1 ? i - 1 : 0, oy = ey == 1 ? j - 1 : 0;
                  const int lx = ex == 1 ? Lx - 1 : 1, ly = ey == 1 ? Ly - 1 : 1;
                  e2 = ex + 3 * ey; o2 = ox + lx * oy; cw = j * WX + i; pstride = lx * ly;
                }
                const int K = L * P + k0 + kk;
                const int ez = K == 0 ? 0 : (K == Lz ? 2 : 1);
                const i64 gi = st27[e2 + 9 * ez] + o2 + (ez == 1 ? (i64)pstride * (K - 1) : 0);
                MFCG_CHECK(gi >= n_int && gi < g.n_dofs && cw >= 0 && cw < PLANE && K >= 0 && K <= Lz);
                pp[c] = MODE == 0 ? src[gi] : Pv[gi];
                mk[c] = g.mask[gi - n_int] & 1;
                dst[c] = (K % RB) * PLANE + cw;
              }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
              if (dst[c] >= 0) ring[dst[c]] = mk[c] ? (T)0 : pp[c];
          }
        }
        // (c) the brick's bottom / top face interiors (first / last layer only): contiguous
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (side == 0 ? (L != 0) : (L != bcz - 1)) continue;
          const i64 fb = st27[side == 0 ? 4 : 22];
          const int slot = ((side == 0 ? 0 : Lz) % RB) * PLANE;
          for (int it = ptid; it < nint2d; it += NT_P) {
            MFCG_CHECK(fb + it >= n_int && fb + it < g.n_dofs);
            const T pv = MODE == 0 ? src[fb + it] : Pv[fb + it];
            const unsigned char mk = g.mask[fb + it - n_int] & 1;
            const int jm = (int)(((unsigned)it * lxm_magic) >> 16);
            const int im = it - jm * lxm;
            ring[slot + (jm + 1) * WX + im + 1] = mk ? (T)0 : pv;
          }
        }
        mbar_arrive(&bars[stage]);  // layer L full
        MFCG_TOC(tp, 1);
      }
      if (!POST_FIRST) do_post();
    }
    if (MODE == 1 && !ONCHIP && PER_BRICK_SUMS) {  // one warp reduction per brick, not per layer
      warp_reduce7(s);
      if ((ptid & 31) == 0)
#pragma unroll
        for (int q = 0; q < 7; ++q) red[pwarp * 7 + q] = s[q];
    }
  } else {
    // ===================== math warps =====================
    // Fixed ownership: TPC threads per cell, thread q of a cell owns lines q, q+TPC, ... of
    // that cell in every sweep of every layer, so all index arithmetic is hoisted.
    constexpr int TPC = Cfg<P, G>::TPC, LPT = (N * N + TPC - 1) / TPC;
    constexpr bool CM = Geo<P, G>::CELL_MINOR;
    constexpr int UNROLL_T = MFCG_UNROLL_T;  // lines of a sweep in flight per thread
    const int cell = CM ? tid % NCELL : tid / TPC, q = CM ? tid / NCELL : tid - cell * TPC;
    // cell-minor: the padding lanes of the last warp own no lines (cell-major: q < TPC by construction)
    const bool has_cell = cell < bcx * bcy && (!CM || q < TPC);
    const int cy = has_cell ? cell / bcx : 0, cx = has_cell ? cell - cy * bcx : 0;
    T* const At = A + cell * TILE;
    T* const Bt = Bs + cell * TILE;
    const T* const ring_cell = ring + cy * P * WX + cx * P;
    if (ONCHIP && (tid & 31) == 0)
      for (int qq = 0; qq < 7; ++qq) red[(tid >> 5) * 7 + qq] = 0.0;
    MFCG_TIC(tc);
    for (int L = 0; L < bcz; ++L) {
      const int stage = L % NS;
      const int s0 = (L * P) % RB;
#ifndef MFCG_LEADER_POLL
      if (L > 0) math_barrier<NT_C>();        // every math thread is done with the previous gather's tiles
      mbar_wait(&bars[stage], (L / NS) & 1);  // layer L full
#else
      // layer L full; the barrier also says every math thread is done with the previous gather's tiles
      if (tid < 32) mbar_wait(&bars[stage], (L / NS) & 1);
      math_barrier<NT_C>();
#endif
      MFCG_TOC(tc, 4);

      if (G >= 1) {
        // ===== general coefficient tensor: 12 sweeps + pointwise flux (operator.py:253-281) =====
        T* const Ct = Bs + NCELL * TILE + cell * TILE;  // third tile of the cell
        // line l of a sweep direction: base offset and element stride inside a tile
        //   x lines (k,j): l*RS, 1;  y lines (k,i): k*N*RS + i, RS;  z lines (j,i): j*RS + i, N*RS
        auto line_base = [&](int dir, int l) {
          const int hi = l / N, lo = l - hi * N;
          return dir == 0 ? hi * PSTR + lo * RS : (dir == 1 ? hi * PSTR + lo : hi * RS + lo);
        };
        constexpr int STR[3] = {1, RS, PSTR};
        // out-of-place or in-place 1D operator on the owned lines of direction dir
        auto sweep = [&](int dir, int kind, bool tr, bool acc, const T* srct, int sstride_unused, T* dstt) {
          (void)sstride_unused;
          if (!has_cell || (MFCG_SKIP & 1)) return;
#pragma unroll 1
          for (int t = 0; t < LPT; ++t) {
            const int l = q + t * TPC;
            if (l >= N * N) break;
            const int base = line_base(dir, l);
            const int str = dir == 0 ? STR[0] : (dir == 1 ? STR[1] : STR[2]);
            T u[N], e[HE], o[HE], se[HE], so[HE], out[N];
#pragma unroll
            for (int i = 0; i < N; ++i) u[i] = srct[base + i * str];
            eo_split<N>(u, e, o);
            if (kind == 0) eo_apply_sym<N>(gen.Se, gen.So, tr, e, o, se, so);
            else eo_apply_anti<N>(gen.Be, gen.Bo, tr, e, o, se, so);
            eo_join<N>(se, so, out);
#pragma unroll
            for (int i = 0; i < N; ++i) {
              if (acc) dstt[base + i * str] += out[i];
              else dstt[base + i * str] = out[i];
            }
          }
        };
        // 1. interpolate to the quadrature points: x from the ring, then y, z in place
        if (has_cell && !(MFCG_SKIP & 1)) {
#pragma unroll 1
          for (int t = 0; t < LPT; ++t) {
            const int l = q + t * TPC;
            if (l >= N * N) break;
            const int k = l / N, j = l - k * N;
            int slot = s0 + k;
            if (slot >= RB) slot -= RB;
            const T* row = ring_cell + slot * PLANE + j * WX;
            T u[N], e[HE], o[HE], se[HE], so[HE], out[N];
#pragma unroll
            for (int i = 0; i < N; ++i) u[i] = row[i];
            eo_split<N>(u, e, o);
            eo_apply_sym<N>(gen.Se, gen.So, false, e, o, se, so);
            eo_join<N>(se, so, out);
#pragma unroll
            for (int i = 0; i < N; ++i) At[k * PSTR + j * RS + i] = out[i];
          }
        }
        if (!ONCHIP) mbar_arrive(&bars[NS + stage]);  // this thread has read its ring rows of layer L
        math_barrier<NT_C>();
        sweep(1, 0, false, false, At, 0, At);
        math_barrier<NT_C>();
        sweep(2, 0, false, false, At, 0, At);
        math_barrier<NT_C>();
        // 2. reference-space gradient at the quadrature points: x -> Bt, y -> Ct (z in registers below)
        sweep(0, 1, false, false, At, 0, Bt);
        sweep(1, 1, false, false, At, 0, Ct);
        math_barrier<NT_C>();
        // 3. per z column: gz, flux = G grad at every point, z part of the transposed gradient
        if (has_cell && !(MFCG_SKIP & 1)) {
          const i64 cellg = ((i64)(mz * g.B[2] + L) * g.cells[1] + (my * g.B[1] + cy)) * g.cells[0] + (mx * g.B[0] + cx);
          constexpr int NQ3 = N * N * N;
#pragma unroll 1
          for (int t = 0; t < LPT; ++t) {
            const int l = q + t * TPC;
            if (l >= N * N) break;
            const int j = l / N, i = l - j * N;
            const int base = j * RS + i;
            T u[N], e[HE], o[HE], se[HE], so[HE], gz[N], fz[N];
#pragma unroll
            for (int k = 0; k < N; ++k) u[k] = At[base + k * PSTR];
            eo_split<N>(u, e, o);
            eo_apply_anti<N>(gen.Be, gen.Bo, false, e, o, se, so);
            eo_join<N>(se, so, gz);
            // on-the-fly geometry: contract the cell's 27 nodes with the x / y basis of this column
            // once (mesh.py:155-174 evaluates the same tri-quadratic map); 27 sums per column
            double colx[9], coly[9], colv[9];
            if (G == 2) {
              const double* nd = reinterpret_cast<const double*>(geo.data) + (i64)cellg * 81;
#pragma unroll
              for (int t9 = 0; t9 < 9; ++t9) { colx[t9] = 0.0; coly[t9] = 0.0; colv[t9] = 0.0; }
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int b3 = 0; b3 < 3; ++b3) {
                  const double vy = (double)gen.qv[j * 3 + b3], dy = (double)gen.qd[j * 3 + b3];
#pragma unroll
                  for (int a3 = 0; a3 < 3; ++a3) {
                    const double vx = (double)gen.qv[i * 3 + a3], dx = (double)gen.qd[i * 3 + a3];
                    const double wx = dx * vy, wy = vx * dy, wv = vx * vy;
                    const double* n3 = nd + 3 * ((c * 3 + b3) * 3 + a3);
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                      colx[c * 3 + d] += n3[d] * wx;
                      coly[c * 3 + d] += n3[d] * wy;
                      colv[c * 3 + d] += n3[d] * wv;
                    }
                  }
                }
            }
#pragma unroll
            for (int k = 0; k < N; ++k) {
              const int qp = (k * N + j) * N + i;
              T G6[6];
              if (G == 1 && geo.kind == 1) {
                const T* gp = reinterpret_cast<const T*>(geo.data) + ((i64)cellg * NQ3 + qp) * 6;
#pragma unroll
                for (int c = 0; c < 6; ++c) G6[c] = gp[c];
              } else {
                double inv[9], jxw, g6d[6];
                if (G == 1) {
                  const T* ip = reinterpret_cast<const T*>(geo.data) + ((i64)cellg * NQ3 + qp) * 9;
#pragma unroll
                  for (int c = 0; c < 9; ++c) inv[c] = (double)ip[c];
                  jxw = (double)reinterpret_cast<const T*>(geo.jxw)[(i64)cellg * NQ3 + qp];
                } else {
                  // J(xi_i, eta_j, zeta_k) from the column's pre-contracted node sums
                  double J[9];
#pragma unroll
                  for (int d = 0; d < 3; ++d) {
                    double jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                      const double vz = (double)gen.qv[k * 3 + c], dz = (double)gen.qd[k * 3 + c];
                      jx += colx[c * 3 + d] * vz;
                      jy += coly[c * 3 + d] * vz;
                      jz += colv[c * 3 + d] * dz;
                    }
                    J[d * 3 + 0] = jx; J[d * 3 + 1] = jy; J[d * 3 + 2] = jz;
                  }
                  const double det = invert3(J, inv);
                  jxw = det * (double)gen.w3[i] * (double)gen.w3[j] * (double)gen.w3[k];
                }
                tensor6(inv, jxw, g6d);
#pragma unroll
                for (int c = 0; c < 6; ++c) G6[c] = (T)g6d[c];
              }
              const T gx = Bt[base + k * PSTR], gy = Ct[base + k * PSTR], gzz = gz[k];
              Bt[base + k * PSTR] = G6[0] * gx + G6[3] * gy + G6[4] * gzz;
              Ct[base + k * PSTR] = G6[3] * gx + G6[1] * gy + G6[5] * gzz;
              fz[k] = G6[4] * gx + G6[5] * gy + G6[2] * gzz;
            }
            eo_split<N>(fz, e, o);
            eo_apply_anti<N>(gen.Be, gen.Bo, true, e, o, se, so);
            eo_join<N>(se, so, u);
#pragma unroll
            for (int k = 0; k < N; ++k) At[base + k * PSTR] = u[k];
          }
        }
        math_barrier<NT_C>();
        // 4. remaining transposed gradient parts accumulate into At, then integrate (S^T) x, y, z
        sweep(0, 1, true, true, Bt, 0, At);
        math_barrier<NT_C>();
        sweep(1, 1, true, true, Ct, 0, At);
        math_barrier<NT_C>();
        sweep(0, 0, true, false, At, 0, At);
        math_barrier<NT_C>();
        sweep(1, 0, true, false, At, 0, At);
        math_barrier<NT_C>();
        sweep(2, 0, true, false, At, 0, At);
        math_barrier<NT_C>();
      } else {
        // ---- x sweep: a = M u, b = gx K u along every x line of the cell
        if (has_cell && !(MFCG_SKIP & 1)) {
  #pragma unroll UNROLL_T
          for (int t = 0; t < LPT; ++t) {
            const int l = LineOrder<N>::x(q + t * TPC, TPC);
            if (l < 0) continue;
            const int k = l / N, j = l - k * N;
            int slot = s0 + k;
            if (slot >= RB) slot -= RB;
            const T* row = ring_cell + slot * PLANE + j * WX;
            T u[N], e[HE], o[HE];
  #pragma unroll
            for (int i = 0; i < N; ++i) u[i] = row[i];
            eo_split<N>(u, e, o);
            T* ao = At + k * PSTR + j * RS;
            T* bo = Bt + k * PSTR + j * RS;
            T se[HE], so[HE], out[N];
  #pragma unroll
            for (int i = 0; i < HE; ++i) { se[i] = 0; so[i] = 0; }
            eo_mul<N>(tab.Me, tab.Mo, e, o, se, so);
            eo_join<N>(se, so, out);
  #pragma unroll
            for (int i = 0; i < N; ++i) ao[i] = out[i];
  #pragma unroll
            for (int i = 0; i < HE; ++i) { se[i] = 0; so[i] = 0; }
            eo_mul<N>(tab.Ke[0], tab.Ko[0], e, o, se, so);
            eo_join<N>(se, so, out);
  #pragma unroll
            for (int i = 0; i < N; ++i) bo[i] = out[i];
          }
        }
        if (!ONCHIP) mbar_arrive(&bars[NS + stage]);  // this thread has read its ring rows of layer L
        MFCG_TOC(tc, 5);
        math_barrier<NT_C>();
        MFCG_TOC(tc, 8);

        // ---- y sweep (in place): c = M a, de = gy K a + M b
        if (has_cell && !(MFCG_SKIP & 1)) {
  #pragma unroll UNROLL_T
          for (int t = 0; t < LPT; ++t) {
            const int l = LineOrder<N>::y(q + t * TPC, TPC);
            if (l < 0) continue;
            const int k = l / N, i = l - k * N;
            T* ac = At + k * PSTR + i;
            T* bc = Bt + k * PSTR + i;
            T a[N], ea[HE], oa[HE], eb[HE], ob[HE];
  #pragma unroll
            for (int j = 0; j < N; ++j) a[j] = ac[j * RS];
            eo_split<N>(a, ea, oa);
  #pragma unroll
            for (int j = 0; j < N; ++j) a[j] = bc[j * RS];
            eo_split<N>(a, eb, ob);
            T se[HE], so[HE], out[N];
  #pragma unroll
            for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
            eo_mul<N>(tab.Ke[1], tab.Ko[1], ea, oa, se, so);  // gy K a
            eo_mul<N>(tab.Me, tab.Mo, eb, ob, se, so);  // + M b
            eo_join<N>(se, so, out);
  #pragma unroll
            for (int j = 0; j < N; ++j) bc[j * RS] = out[j];
  #pragma unroll
            for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
            eo_mul<N>(tab.Me, tab.Mo, ea, oa, se, so);  // c = M a
            eo_join<N>(se, so, out);
  #pragma unroll
            for (int j = 0; j < N; ++j) ac[j * RS] = out[j];
          }
        }
        MFCG_TOC(tc, 6);
        math_barrier<NT_C>();
        MFCG_TOC(tc, 8);

        // ---- z sweep: out = M de + gz K c, written over c
        if (has_cell && !(MFCG_SKIP & 1)) {
  #pragma unroll UNROLL_T
          for (int t = 0; t < LPT; ++t) {
            const int l = LineOrder<N>::z(q + t * TPC, TPC);
            if (l < 0) continue;
            const int j = l / N, i = l - j * N;
            T* ac = At + j * RS + i;
            const T* bc = Bt + j * RS + i;
            T a[N], ec[HE], oc[HE], ed[HE], od[HE];
  #pragma unroll
            for (int k = 0; k < N; ++k) a[k] = ac[k * PSTR];
            eo_split<N>(a, ec, oc);
  #pragma unroll
            for (int k = 0; k < N; ++k) a[k] = bc[k * PSTR];
            eo_split<N>(a, ed, od);
            T se[HE], so[HE], out[N];
  #pragma unroll
            for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
            eo_mul<N>(tab.Ke[2], tab.Ko[2], ec, oc, se, so);  // gz K c
            eo_mul<N>(tab.Me, tab.Mo, ed, od, se, so);  // + M de
            eo_join<N>(se, so, out);
  #pragma unroll
            for (int k = 0; k < N; ++k) ac[k * PSTR] = out[k];
          }
        }
        MFCG_TOC(tc, 7);
        math_barrier<NT_C>();
        MFCG_TOC(tc, 8);

      }

      // ---- gather the cells' contributions per lattice point, finish the planes
      double s[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int rem = tid; rem < ((MFCG_SKIP & 2) ? 0 : fp); rem += NT_C) {
        MFCG_CHECK(!USE_GTAB || rem < Geo<P, G>::GTAB_N);
        const uint2 d = USE_GTAB ? gtab[rem] : gather_descriptor(rem);
        const int base = (int)(d.x & 16383u), cw = (int)(d.y & 1023u), o2 = (int)((d.y >> 10) & 4095u);
        if (!ONCHIP && ((d.x >> 14) & 31u) == 1u) {
          // strictly inside one cell in x and y: one contribution per plane, brick-interior DoFs
          const T* a = A + base;
          const i64 gi0 = st27[13] + o2 + (i64)nint2d_c * (L * P - 1);
          MFCG_CHECK(base + P * PSTR < NCELL * TILE && cw < PLANE);
          {
            const T sum = a[0] + carry[cw];
            if (L == 0) atomicAdd(&V[st27[4] + o2], sum);  // the brick's bottom face is shared
            else { MFCG_CHECK(gi0 >= 0 && gi0 < n_int); V[gi0] = sum; }
          }
#pragma unroll
          for (int k = 1; k < P; ++k) {
            MFCG_CHECK(gi0 + (i64)k * nint2d_c >= 0 && gi0 + (i64)k * nint2d_c < n_int);
            V[gi0 + (i64)k * nint2d_c] = a[k * PSTR];
          }
          if (L < bcz - 1) carry[cw] = a[P * PSTR];
          else atomicAdd(&V[st27[22] + o2], a[P * PSTR]);  // top face
          continue;
        }
        const bool edge = (d.x >> 18) & 1u;
        const int e2 = (int)((d.x >> 19) & 15u);
        const unsigned sel = d.y >> 22;
        const int pstride = ((sel & 1u) ? Lx - 1 : 1) * ((sel & 2u) ? Ly - 1 : 1);
        // offsets of the (up to four) cell-tile entries holding this point
        const int o11 = (d.x & (1u << 14)) ? base : -1;
        const int o10 = (d.x & (1u << 15)) ? base - TILE + P : -1;
        const int o01 = (d.x & (1u << 16)) ? base - bcx * TILE + P * RS : -1;
        const int o00 = (d.x & (1u << 17)) ? base - (bcx + 1) * TILE + P * RS + P : -1;
#pragma unroll
        for (int k = 0; k <= P; ++k) {
          T sum = 0;
          if (o00 >= 0) sum += A[o00 + k * PSTR];
          if (o01 >= 0) sum += A[o01 + k * PSTR];
          if (o10 >= 0) sum += A[o10 + k * PSTR];
          if (o11 >= 0) sum += A[o11 + k * PSTR];
          if (k == 0) sum += carry[cw];
          if (k == P && L < bcz - 1) {
            carry[cw] = sum;
            continue;
          }
          const int K = L * P + k;
          const int ez = K == 0 ? 0 : (K == Lz ? 2 : 1);
          const i64 gi = st27[e2 + 9 * ez] + o2 + (ez == 1 ? (i64)pstride * (K - 1) : 0);
          // constrained rows receive garbage here; k_post / k_surface_fix restore v_c = p_c
          MFCG_CHECK((edge || ez != 1) ? (gi >= n_int && gi < g.n_dofs) : (gi >= 0 && gi < n_int));
          MFCG_CHECK(o11 < NCELL * TILE && o10 < NCELL * TILE && o01 < NCELL * TILE && o00 < NCELL * TILE);
          if (!(edge || ez != 1)) {
            V[gi] = sum;
            if (ONCHIP) {  // post on values that never left the SM (solvers.py:692-698)
              int slot = s0 + k;
              if (slot >= RB) slot -= RB;
              const int ro = slot * PLANE + cw;
              const double r = (double)Rring[ro], m = (double)Mring[ro], p = (double)ring[ro], v = (double)sum;
              const double mr = m * r, mv = m * v;
              s[0] += r * r; s[1] += p * v; s[2] += r * v; s[3] += v * v;
              s[4] += r * mr; s[5] += r * mv; s[6] += v * mv;
            }
          } else {
            atomicAdd(&V[gi], sum);
          }
        }
      }
      if (ONCHIP) {
        warp_reduce7(s);
        if ((tid & 31) == 0)
#pragma unroll
          for (int qq = 0; qq < 7; ++qq) red[(tid >> 5) * 7 + qq] += s[qq];
      }
      if (ONCHIP) mbar_arrive(&bars[NS + stage]);  // the on-chip post reads the ring in the gather
      mbar_arrive(&bars[2 * NS + stage]);  // v of layer L stored (orders the v stores before the post loads)
      MFCG_TOC(tc, 9);
    }
  }
#ifdef MFCG_TIMING
  __syncthreads();
  if (threadIdx.x < 16 && tcnt[threadIdx.x]) atomicAdd(&g_phase_cycles[threadIdx.x], tcnt[threadIdx.x]);
#endif
  if (MODE == 1) {
    // block sums: the memory warps' slots, added in a fixed order (deterministic)
    __syncthreads();
    if (tid < 7) {
      double acc = 0.0;
      if (ONCHIP) {
        for (int w = 0; w < NT_C / 32; ++w) acc += red[w * 7 + tid];
      } else {
        for (int w = 0; w < NT_P / 32; ++w) acc += red[w * 7 + tid];
      }
      partials[(i64)b * 8 + tid] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// Range kernels over [lo, hi) in brick numbering.

// dst = 0 on the shared range before the atomic accumulation (operator.py:334-335)
template <typename T>
__global__ void k_surface_init(BrickGrid g, T* __restrict__ dst) {
  const i64 n_sh = g.n_dofs - g.n_int;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n_sh; i += (i64)gridDim.x * blockDim.x)
    dst[g.n_int + i] = (T)0;
}

// constrained rows are identity: dst[c] = src[c] (operator.py:359-360)
template <typename T>
__global__ void k_surface_fix(BrickGrid g, const T* __restrict__ src, T* __restrict__ dst) {
  const i64 n_sh = g.n_dofs - g.n_int;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n_sh; i += (i64)gridDim.x * blockDim.x)
    if (g.mask[i] & 1) dst[g.n_int + i] = src[g.n_int + i];
}

// merged-CG "pre" (solvers.py:660-690); with init_v also zeroes v for the
// atomic accumulation of the brick kernel.
template <typename T>
__global__ void k_pre(BrickGrid g, i64 lo, i64 hi, int init_v, T* __restrict__ R, T* __restrict__ Pv,
                      T* __restrict__ V, T* __restrict__ X, const T* __restrict__ Minv,
                      const SolveState* __restrict__ st) {
  if (!st->active) return;
  const T am1 = (T)st->am1, bm1 = (T)st->bm1, xc1 = (T)st->xc1, xc2 = (T)st->xc2;
  const int xmode = st->xmode;
  constexpr int U = 4;  // independent loads in flight per thread
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i0 = lo + blockIdx.x * (i64)blockDim.x + threadIdx.x; i0 < hi; i0 += U * stride) {
    T r[U], p[U], v[U], m[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 i = i0 + u * stride;
      if (i < hi) {
        r[u] = R[i]; p[u] = Pv[i]; v[u] = V[i]; m[u] = Minv[i];
        if (xmode) x[u] = X[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 i = i0 + u * stride;
      if (i >= hi) break;
      if (xmode) {
        if (xmode == 2) x[u] += xc1 * p[u] + xc2 * (p[u] - m[u] * r[u]);
        else x[u] += xc1 * p[u];
        X[i] = x[u];
      }
      r[u] -= am1 * v[u];
      p[u] = m[u] * r[u] + bm1 * p[u];
      R[i] = r[u];
      Pv[i] = p[u];
      if (init_v) V[i] = (T)0;
    }
  }
}

// merged-CG "post": the seven sums (solvers.py:112-127, 692-698)
template <typename T>
__global__ void k_post(BrickGrid g, i64 lo, i64 hi, int fix_constrained, const T* __restrict__ R,
                       const T* __restrict__ Pv, T* __restrict__ V, const T* __restrict__ Minv,
                       const SolveState* __restrict__ st, double* __restrict__ partials) {
  __shared__ double red[7 * 32];
  if (!st->active) return;
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  constexpr int U = 4;  // independent loads in flight per thread
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i0 = lo + blockIdx.x * (i64)blockDim.x + threadIdx.x; i0 < hi; i0 += U * stride) {
    T rr[U], pp[U], mm[U], vv[U];
    unsigned char ff[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 i = i0 + u * stride;
      ff[u] = 0;
      if (i < hi) {
        rr[u] = R[i]; pp[u] = Pv[i]; mm[u] = Minv[i]; vv[u] = V[i];
        if (i >= g.n_int) ff[u] = g.mask[i - g.n_int];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 i = i0 + u * stride;
      if (i >= hi) break;
      const double r = (double)rr[u], p = (double)pp[u], m = (double)mm[u];
      double v = (double)vv[u];
      const unsigned char flag = ff[u];
      if (fix_constrained && (flag & 1)) {  // identity row: v_c = p_c
        v = p;
        V[i] = (T)p;
      }
      if (flag & 2) continue;  // ghost copy of the lower slab's plane: counted there
      const double mr = m * r, mv = m * v;
      s[0] += r * r; s[1] += p * v; s[2] += r * v; s[3] += v * v;
      s[4] += r * mr; s[5] += r * mv; s[6] += v * mv;
    }
  }
  block_reduce7_store(s, red, partials + (i64)blockIdx.x * 8);
}

// x catch-up after the loop (solvers.py:771-782)
template <typename T>
__global__ void k_finalize_x(i64 n, T* __restrict__ X, const T* __restrict__ Pv, const T* __restrict__ R,
                             const T* __restrict__ Minv, const SolveState* __restrict__ st) {
  const int k = st->k;
  if (k <= 0) return;
  const T a1 = (T)st->am1;
  const bool simple = st->force_x || (k & 1) || st->am2 == 0.0 || st->bm2 == 0.0;
  const T c2 = simple ? (T)0 : (T)(st->am2 / st->bm2);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const T p = Pv[i];
    X[i] += simple ? a1 * p : a1 * p + c2 * (p - Minv[i] * R[i]);
  }
}

// Deterministic sum of `rows` partial rows (stride 8) into out[0..cols)
__device__ __forceinline__ void reduce_rows(const double* __restrict__ partials, int rows, int cols, double* out,
                                            double* red /* blockDim.x * cols? no: 8*32 */) {
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int r = threadIdx.x; r < rows; r += blockDim.x)
    for (int q = 0; q < cols; ++q) s[q] += partials[(i64)r * 8 + q];
  warp_reduce7(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0)
    for (int q = 0; q < 7; ++q) red[w * 7 + q] = s[q];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < cols; ++q) {
      double acc = 0.0;
      for (int i = 0; i < nw; ++i) acc += red[i * 7 + q];
      out[q] = acc;
    }
  __syncthreads();
}

// Scalar step of the merged iteration (solvers.py:706-764) on the seven reduced sums.
__device__ __forceinline__ void merged_scalar_step(const double* sums, SolveState* st, double* __restrict__ history) {
  const double gamma = sums[0], a = sums[1], bb = sums[2], cc = sums[3], d = sums[4], e = sums[5], f = sums[6];
  const int k = st->k + 1;
  const bool fixed = st->fixed != 0;
  double alpha = 0.0, beta = 0.0, residual = st->residual;
  bool stop = false;
  if (st->stagnant) {
    residual = sqrt(gamma) / st->bnorm;
  } else if (gamma == 0.0) {
    residual = 0.0;
    if (fixed) st->stagnant = 1;
    else { st->converged = 1; stop = true; }
  } else if (st->has_prec && d <= 0.0) {
    st->breakdown = 2; st->breakdown_value = d; st->breakdown_iteration = k; st->active = 0;
    return;
  } else if (a <= 0.0) {
    if (fixed && residual < st->tol) st->stagnant = 1;
    else { st->breakdown = 1; st->breakdown_value = a; st->breakdown_iteration = k; st->active = 0; return; }
  } else {
    alpha = d / a;
    beta = (d - 2.0 * alpha * e + alpha * alpha * f) / d;
    const double stop_sq = gamma - 2.0 * alpha * bb + alpha * alpha * cc;
    residual = sqrt(stop_sq > 0.0 ? stop_sq : 0.0) / st->bnorm;
    if (beta <= 0.0 && fixed) {
      if (residual < st->tol) st->stagnant = 1;
      else { st->breakdown = 3; st->breakdown_value = beta; st->breakdown_iteration = k; st->active = 0; return; }
    }
  }
  history[(i64)(k - 1) * 4 + 0] = alpha;
  history[(i64)(k - 1) * 4 + 1] = beta;
  history[(i64)(k - 1) * 4 + 2] = gamma;
  history[(i64)(k - 1) * 4 + 3] = residual;
  st->am2 = st->am1; st->bm2 = st->bm1;
  st->am1 = alpha; st->bm1 = beta;
  st->k = k;
  st->residual = residual;
  if (!fixed && residual < st->tol) { st->converged = 1; stop = true; }
  if (stop || k >= st->limit) st->active = 0;
  // x catch-up of the next pre (iteration k+1), solvers.py:661-677
  const int kn = k + 1;
  const bool live = st->am1 != 0.0 || st->am2 != 0.0;
  int xmode = 0;
  if (kn > 1 && live && (st->force_x || (kn & 1))) {
    if (st->force_x) xmode = 1;
    else if (st->am2 != 0.0 && st->bm2 != 0.0) { xmode = 2; st->xc2 = st->am2 / st->bm2; }
    else xmode = 1;
    st->xc1 = st->am1;
  }
  st->xmode = xmode;
}

// one block: reduce the per-block partial rows, then the scalar step
static __global__ void k_scalar_merged(const double* __restrict__ partials, int rows, SolveState* st,
                                       double* __restrict__ history) {
  __shared__ double red[7 * 32];
  __shared__ double sums[8];
  if (!st->active) return;
  reduce_rows(partials, rows, 7, sums, red);
  if (threadIdx.x != 0) return;
#if MFCG_SKIP || defined(MFCG_B2_SKIP_ANY)
  // timing experiments only: keep iterating on garbage
  sums[0] = sums[1] = sums[3] = sums[4] = sums[6] = 1.0; sums[2] = sums[5] = 0.25;
#endif
  merged_scalar_step(sums, st, history);
}

// slab runs: the sums arrive already reduced over all slabs / ranks
static __global__ void k_scalar_merged_sums(const double* __restrict__ sums, SolveState* st,
                                            double* __restrict__ history) {
  if (!st->active || threadIdx.x != 0) return;
  merged_scalar_step(sums, st, history);
}

// out[0..cols) = deterministic sum of the partial rows; acc != 0: add to out instead of overwriting
static __global__ void k_reduce_partials(const double* __restrict__ partials, int rows, int cols, int acc,
                                         double* __restrict__ out) {
  __shared__ double red[7 * 32];
  __shared__ double sums[8];
  reduce_rows(partials, rows, cols, sums, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < cols; ++q) out[q] = acc ? out[q] + sums[q] : sums[q];
}

// ---------------------------------------------------------------------------
// Standard (unfused) CG / PCG: one kernel per vector region of the reference
// (solvers.py:296-336), scalars stay on the device.

template <typename T>
__global__ void k_dot(i64 n, const T* __restrict__ a, const T* __restrict__ b, const SolveState* st,
                      double* __restrict__ partials) {
  __shared__ double red[7 * 32];
  if (st && !st->active) return;
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    s[0] += (double)a[i] * (double)b[i];
  block_reduce7_store(s, red, partials + (i64)blockIdx.x * 8);
}

// r = b, z = M r, p = z (or p = r), partial sums of r.z (col 0) and r.r (col 1)
template <typename T>
__global__ void k_std_init(i64 n, const T* __restrict__ B, const T* __restrict__ Minv, T* __restrict__ R,
                           T* __restrict__ Z, T* __restrict__ Pv, T* __restrict__ X, double* __restrict__ partials) {
  __shared__ double red[7 * 32];
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const T r = B[i];
    const T z = Minv ? Minv[i] * r : r;
    R[i] = r;
    if (Minv) Z[i] = z;
    Pv[i] = z;
    X[i] = (T)0;
    s[0] += (double)r * (double)z;
    s[1] += (double)r * (double)r;
  }
  block_reduce7_store(s, red, partials + (i64)blockIdx.x * 8);
}

static __global__ void k_std_init_scalar(const double* __restrict__ partials, int rows, SolveState* st) {
  __shared__ double red[7 * 32];
  __shared__ double sums[8];
  reduce_rows(partials, rows, 2, sums, red);
  if (threadIdx.x != 0) return;
  st->gamma = sums[0];
  st->residual = sqrt(sums[1]) / st->bnorm;
}

// alpha = gamma / (p.v) with the breakdown rule of solvers.py:302-310
static __global__ void k_std_alpha(const double* __restrict__ partials, int rows, SolveState* st) {
  __shared__ double red[7 * 32];
  __shared__ double sums[8];
  if (!st->active) return;
  reduce_rows(partials, rows, 1, sums, red);
  if (threadIdx.x != 0) return;
  const double a = sums[0];
  if (a <= 0.0) {
    if (st->fixed && st->residual < st->tol) st->alpha = 0.0;
    else { st->breakdown = 1; st->breakdown_value = a; st->breakdown_iteration = st->k + 1; st->active = 0; }
  } else {
    st->alpha = st->gamma / a;
  }
}

// y += sign * alpha * x
template <typename T>
__global__ void k_std_axpy(i64 n, T* __restrict__ y, const T* __restrict__ x, double sign, const SolveState* st) {
  if (!st->active) return;
  const T al = (T)(sign * st->alpha);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    y[i] += al * x[i];
}

template <typename T>
__global__ void k_std_prec(i64 n, T* __restrict__ Z, const T* __restrict__ Minv, const T* __restrict__ R,
                           const SolveState* st) {
  if (!st->active) return;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    Z[i] = Minv[i] * R[i];
}

// beta, residual, history (solvers.py:317-333); rr_partials: r.r, rz_partials: r.z (PCG only)
static __global__ void k_std_beta(const double* __restrict__ rr_partials, const double* __restrict__ rz_partials,
                           int rows, SolveState* st, double* __restrict__ history) {
  __shared__ double red[7 * 32];
  __shared__ double sums[8];
  __shared__ double sums2[8];
  if (!st->active) return;
  reduce_rows(rr_partials, rows, 1, sums, red);
  if (rz_partials) reduce_rows(rz_partials, rows, 1, sums2, red);
  if (threadIdx.x != 0) return;
  const double rr = sums[0];
  const double gamma_new = rz_partials ? sums2[0] : rr;
  const double residual = sqrt(rr) / st->bnorm;
  const double beta = st->gamma > 0.0 ? gamma_new / st->gamma : 0.0;
  const int k = st->k + 1;
  history[(i64)(k - 1) * 4 + 0] = st->alpha;
  history[(i64)(k - 1) * 4 + 1] = beta;
  history[(i64)(k - 1) * 4 + 2] = st->gamma;
  history[(i64)(k - 1) * 4 + 3] = residual;
  st->gamma = gamma_new;
  st->beta = beta;
  st->residual = residual;
  st->k = k;
  if (!st->fixed && residual < st->tol) { st->converged = 1; st->active = 0; }
  if (k >= st->limit) st->active = 0;
}

// slab runs: sums[0] = r.r, sums[1] = r.z already reduced over all slabs / ranks
static __global__ void k_std_beta_sums(const double* __restrict__ sums, int prec, SolveState* st,
                                       double* __restrict__ history) {
  if (!st->active || threadIdx.x != 0) return;
  const double rr = sums[0];
  const double gamma_new = prec ? sums[1] : rr;
  const double residual = sqrt(rr) / st->bnorm;
  const double beta = st->gamma > 0.0 ? gamma_new / st->gamma : 0.0;
  const int k = st->k + 1;
  history[(i64)(k - 1) * 4 + 0] = st->alpha;
  history[(i64)(k - 1) * 4 + 1] = beta;
  history[(i64)(k - 1) * 4 + 2] = st->gamma;
  history[(i64)(k - 1) * 4 + 3] = residual;
  st->gamma = gamma_new;
  st->beta = beta;
  st->residual = residual;
  st->k = k;
  if (!st->fixed && residual < st->tol) { st->converged = 1; st->active = 0; }
  if (k >= st->limit) st->active = 0;
}

// p = beta p + z.  Runs even on the iteration that hit the limit in the
// reference (solvers.py:334-335 executes unless the loop broke on convergence);
// p is not observable afterwards, so skipping it when inactive is equivalent.
template <typename T>
__global__ void k_std_update_p(i64 n, T* __restrict__ Pv, const T* __restrict__ Z, const SolveState* st) {
  if (!st->active) return;
  const T be = (T)st->beta;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    Pv[i] = be * Pv[i] + Z[i];
}

// ---------------------------------------------------------------------------
// Numbering helpers

struct LatticeMap {
  int p, cells[3], B[3], mb[3];
  const i64* ent_start;
};

__device__ __forceinline__ void seg_of(int I, int p, int B, int ncell, int mbd, int& s, int& o, int& len) {
  const int W = p * B;
  int m = I / W, rem = I - m * W;
  if (m == mbd) { m = mbd - 1; rem = W; }
  int bc = ncell - m * B;
  if (bc > B) bc = B;
  const int L = p * bc;
  if (rem == 0) { s = 2 * m; o = 0; len = 1; }
  else if (rem == L) { s = 2 * m + 2; o = 0; len = 1; }
  else { s = 2 * m + 1; o = rem - 1; len = L - 1; }
}

// lattice point (I,J,K) of the rank's mesh -> index in brick numbering
__device__ __forceinline__ i64 lattice_to_dev(const BrickGrid& g, int I, int J, int K) {
  int sx, ox, lx, sy, oy, ly, sz, oz, lz;
  seg_of(I, g.p, g.B[0], g.cells[0], g.mb[0], sx, ox, lx);
  seg_of(J, g.p, g.B[1], g.cells[1], g.mb[1], sy, oy, ly);
  seg_of(K, g.p, g.B[2], g.cells[2], g.mb[2], sz, oz, lz);
  (void)lz;
  const i64 e = ((i64)sz * (2 * g.mb[1] + 1) + sy) * (2 * g.mb[0] + 1) + sx;
  return g.ent_start[e] + ox + (i64)lx * (oy + (i64)ly * oz);
}

// perm[user] = device index, from the caller's 27 block starts per cell
// (dofs.py:119-135 expansion rule) and the structured cell position.
static __global__ void k_build_perm(BrickGrid g, const int* __restrict__ blocks, i64 n_cells, int* __restrict__ perm) {
  const int p = g.p, n = p + 1, npc = n * n * n;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < n_cells * npc; t += (i64)gridDim.x * blockDim.x) {
    const i64 cell = t / npc;
    const int node = (int)(t - cell * npc);
    const int i = node % n, j = (node / n) % n, k = node / (n * n);
    const int sx = i == 0 ? 0 : (i == p ? 2 : 1), sy = j == 0 ? 0 : (j == p ? 2 : 1), sz = k == 0 ? 0 : (k == p ? 2 : 1);
    const int cxo = sx == 1 ? i - 1 : 0, cyo = sy == 1 ? j - 1 : 0, czo = sz == 1 ? k - 1 : 0;
    const int mxe = sx == 1 ? p - 1 : 1, mye = sy == 1 ? p - 1 : 1;
    const i64 user = (i64)blocks[cell * 27 + sx + 3 * sy + 9 * sz] + cxo + mxe * (cyo + mye * czo);
    const int cx = (int)(cell % g.cells[0]), cy = (int)((cell / g.cells[0]) % g.cells[1]),
              cz = (int)(cell / ((i64)g.cells[0] * g.cells[1]));
    perm[user] = (int)lattice_to_dev(g, cx * p + i, cy * p + j, cz * p + k);
  }
}

// Caller numbering -> brick numbering.  The caller interleaves the components of a node
// (dofs.py:229-236: index = node * C + c); the device keeps one scalar field per component,
// dev[c * cs + perm[node]] (cs >= n: component stride).  `usr_comp` == 1 replicates a per-node scalar (the Jacobi diagonal,
// operator.py:92-94) into all C fields.
template <typename T>
__global__ void k_to_device_order(i64 n, int C, i64 cs, int usr_comp, const int* __restrict__ perm,
                                  const double* __restrict__ usr, T* __restrict__ dev) {
  const i64 total = n * C;
  for (i64 u = blockIdx.x * (i64)blockDim.x + threadIdx.x; u < total; u += (i64)gridDim.x * blockDim.x) {
    const i64 node = u / C;
    const int c = (int)(u - node * C);
    dev[c * cs + perm[node]] = (T)(usr_comp == 1 ? usr[node] : usr[u]);
  }
}

// usr[node * C + c] = (double) dev[c * cs + perm[node]]
template <typename T>
__global__ void k_to_user_order(i64 n, int C, i64 cs, const int* __restrict__ perm, const T* __restrict__ dev,
                                double* __restrict__ usr) {
  const i64 total = n * C;
  for (i64 u = blockIdx.x * (i64)blockDim.x + threadIdx.x; u < total; u += (i64)gridDim.x * blockDim.x) {
    const i64 node = u / C;
    const int c = (int)(u - node * C);
    usr[u] = (double)dev[c * cs + perm[node]];
  }
}

static __global__ void k_mark_constrained(i64 k, int C, const i64* __restrict__ constrained, const int* __restrict__ perm,
                                   i64 n_int, unsigned char* __restrict__ mask, int* __restrict__ error) {
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < k; t += (i64)gridDim.x * blockDim.x) {
    const i64 d = perm[constrained[t] / C];
    if (d < n_int) *error = 1;  // a constrained DoF strictly inside a brick: not a boundary constraint
    else mask[d - n_int] |= 1;
  }
}

// ---------------------------------------------------------------------------
// z-slab decomposition: neighbouring slabs share one lattice plane; both hold it,
// the lower slab owns it for the dot products.  buf[J * NX + I] <-> vector entry of lattice point
// (I, J, K) of this slab in brick numbering.
template <typename T>
__global__ void k_plane_pack(BrickGrid g, int K, const T* __restrict__ vec, T* __restrict__ buf) {
  const int NX = g.cells[0] * g.p + 1, NY = g.cells[1] * g.p + 1;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < (i64)NX * NY; t += (i64)gridDim.x * blockDim.x) {
    const int J = (int)(t / NX), I = (int)(t - (i64)J * NX);
    buf[t] = vec[lattice_to_dev(g, I, J, K)];
  }
}
template <typename T>
__global__ void k_plane_add(BrickGrid g, int K, T* __restrict__ vec, const T* __restrict__ buf) {
  const int NX = g.cells[0] * g.p + 1, NY = g.cells[1] * g.p + 1;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < (i64)NX * NY; t += (i64)gridDim.x * blockDim.x) {
    const int J = (int)(t / NX), I = (int)(t - (i64)J * NX);
    vec[lattice_to_dev(g, I, J, K)] += buf[t];
  }
}
// flag the slab's bottom plane as a ghost copy (bit 1)
static __global__ void k_mark_ghost_plane(BrickGrid g, int K, unsigned char* __restrict__ mask) {
  const int NX = g.cells[0] * g.p + 1, NY = g.cells[1] * g.p + 1;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < (i64)NX * NY; t += (i64)gridDim.x * blockDim.x) {
    const int J = (int)(t / NX), I = (int)(t - (i64)J * NX);
    mask[lattice_to_dev(g, I, J, K) - g.n_int] |= 2;
  }
}
// partial sums of a.b over the DoFs this slab owns
template <typename T>
__global__ void k_dot_owned(BrickGrid g, const T* __restrict__ a, const T* __restrict__ b,
                            double* __restrict__ partials) {
  __shared__ double red[7 * 32];
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < g.n_dofs; i += (i64)gridDim.x * blockDim.x) {
    if (i >= g.n_int && (g.mask[i - g.n_int] & 2)) continue;
    s[0] += (double)a[i] * (double)b[i];
  }
  block_reduce7_store(s, red, partials + (i64)blockIdx.x * 8);
}
// standard (P)CG on a slab: r = b, z = M r, p = z, x = 0; sums of r.z (col 0) and r.r (col 1) over owned DoFs
template <typename T>
__global__ void k_std_init_owned(BrickGrid g, const T* __restrict__ B, const T* __restrict__ Minv, T* __restrict__ R,
                                 T* __restrict__ Z, T* __restrict__ Pv, T* __restrict__ X, double* __restrict__ partials) {
  __shared__ double red[7 * 32];
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < g.n_dofs; i += (i64)gridDim.x * blockDim.x) {
    const T r = B[i];
    const T z = Minv ? Minv[i] * r : r;
    R[i] = r;
    if (Minv) Z[i] = z;
    Pv[i] = z;
    X[i] = (T)0;
    if (i >= g.n_int && (g.mask[i - g.n_int] & 2)) continue;  // ghost copy: counted by the lower slab
    s[0] += (double)r * (double)z;
    s[1] += (double)r * (double)r;
  }
  block_reduce7_store(s, red, partials + (i64)blockIdx.x * 8);
}

// state for a slab run is written by the host; this sets the norm all slabs share
static __global__ void k_set_bnorm(SolveState* st, const double* __restrict__ sums) { st->bnorm = sqrt(sums[0]); }

// ---------------------------------------------------------------------------
// Jacobi diagonal, GL collocation, affine geometry (operator.py:380-418):
// diag_loc[k,j,i] = gx w_k w_j dd_i + gy w_k w_i dd_j + gz w_j w_i dd_k,
// dd_i = sum_q w_q D[q,i]^2, g_d = det J / h_d^2.
struct DiagTables {
  double w[9], dd[9], g[3];
};

static __global__ void k_diag_affine(BrickGrid g, DiagTables t, i64 n_cells, double* __restrict__ diag) {
  const int p = g.p, n = p + 1, npc = n * n * n;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < n_cells * npc; q += (i64)gridDim.x * blockDim.x) {
    const i64 cell = q / npc;
    const int node = (int)(q - cell * npc);
    const int i = node % n, j = (node / n) % n, k = node / (n * n);
    const int cx = (int)(cell % g.cells[0]), cy = (int)((cell / g.cells[0]) % g.cells[1]),
              cz = (int)(cell / ((i64)g.cells[0] * g.cells[1]));
    const double val = t.g[0] * t.w[k] * t.w[j] * t.dd[i] + t.g[1] * t.w[k] * t.w[i] * t.dd[j] +
                       t.g[2] * t.w[j] * t.w[i] * t.dd[k];
    atomicAdd(&diag[lattice_to_dev(g, cx * p + i, cy * p + j, cz * p + k)], val);
  }
}

// diag -> 1/diag with constrained entries 1; flags non-positive / non-finite
static __global__ void k_diag_invert(BrickGrid g, double* __restrict__ diag, int* __restrict__ error) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < g.n_dofs; i += (i64)gridDim.x * blockDim.x) {
    double d = diag[i];
    if (i >= g.n_int && (g.mask[i - g.n_int] & 1)) d = 1.0;
    if (!(d > 0.0) || isinf(d)) *error = 1;
    diag[i] = 1.0 / d;
  }
}

template <typename TO, typename TI>
__global__ void k_convert(i64 n, const TI* __restrict__ in, TO* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = (TO)in[i];
}

template <typename T>
__global__ void k_fill(i64 n, T* __restrict__ out, T value) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = value;
}


// ---------------------------------------------------------------------------
// Geometry set-up on the device (mesh.py:126-174, 194-252).  One block per cell: the 27
// tri-quadratic nodes of the cell are the sine-bump map of the {0,1/2,1}^3 lattice
// (mesh.py:73-80), then every thread evaluates Jacobians at tensor points.
struct GeoMesh {
  int cells[3];   // cells of this slab
  int z0;         // first global cell layer of the slab
  double h[3], ext[3], amp;  // ext: extents of the whole mesh
};
struct PointTab {   // quadratic basis on {0,1/2,1} at up to 10 1D points, and their weights
  double qv[30], qd[30], w[10];
  int n;
};

__device__ __forceinline__ void cell_nodes_to_smem(const GeoMesh& gm, i64 cell, double* nodes /*[81]*/) {
  const int cx = (int)(cell % gm.cells[0]), cy = (int)((cell / gm.cells[0]) % gm.cells[1]),
            cz = (int)(cell / ((i64)gm.cells[0] * gm.cells[1])) + gm.z0;
  const double kPi = 3.14159265358979323846;
  if (threadIdx.x < 27) {
    const int a = threadIdx.x % 3, b = (threadIdx.x / 3) % 3, c = threadIdx.x / 9;
    const double X = cx * gm.h[0] + (0.5 * a) * gm.h[0], Y = cy * gm.h[1] + (0.5 * b) * gm.h[1],
                 Z = cz * gm.h[2] + (0.5 * c) * gm.h[2];
    double bump = 0.0;
    if (gm.amp != 0.0)
      bump = gm.amp * (sin(kPi * X / gm.ext[0]) * sin(kPi * Y / gm.ext[1]) * sin(kPi * Z / gm.ext[2]));
    nodes[threadIdx.x * 3 + 0] = X + bump;
    nodes[threadIdx.x * 3 + 1] = Y + bump;
    nodes[threadIdx.x * 3 + 2] = Z + bump;
  }
}

// kind 1: a = final tensor [cell][q][6]; kind 2: a = inverse Jacobian [cell][q][9], b = jxw [cell][q];
// kind 3: a = nodes [cell][27][3] (always double).  error: 1 if some det J <= 0 (mesh.py:171-172).
template <typename T>
__global__ void k_geometry(GeoMesh gm, PointTab pt, i64 n_cells, int kind, T* __restrict__ a, T* __restrict__ b,
                           double* __restrict__ nodes_out, int* __restrict__ error) {
  __shared__ double nodes[81];
  const int n = pt.n, nq3 = n * n * n;
  for (i64 cell = blockIdx.x; cell < n_cells; cell += gridDim.x) {
    __syncthreads();
    cell_nodes_to_smem(gm, cell, nodes);
    __syncthreads();
    if (kind == 3) {
      for (int t = threadIdx.x; t < 81; t += blockDim.x) nodes_out[cell * 81 + t] = nodes[t];
      continue;
    }
    for (int q = threadIdx.x; q < nq3; q += blockDim.x) {
      const int i = q % n, j = (q / n) % n, k = q / (n * n);
      double J[9], inv[9];
      jacobian27(nodes, pt.qv + 3 * i, pt.qd + 3 * i, pt.qv + 3 * j, pt.qd + 3 * j, pt.qv + 3 * k, pt.qd + 3 * k, J);
      const double det = invert3(J, inv);
      if (!(det > 0.0)) *error = 1;
      const double jxw = det * (pt.w[k] * pt.w[j] * pt.w[i]);
      if (kind == 1) {
        double g6[6];
        tensor6(inv, jxw, g6);
        for (int c = 0; c < 6; ++c) a[(cell * nq3 + q) * 6 + c] = (T)g6[c];
      } else {
        for (int c = 0; c < 9; ++c) a[(cell * nq3 + q) * 9 + c] = (T)inv[c];
        b[cell * nq3 + q] = (T)jxw;
      }
    }
  }
}

// Jacobi diagonal on general geometry (operator.py:380-418): GL collocation, coefficient tensor of
// the tri-quadratic map at the (p+1)^3 Gauss-Lobatto points of every cell.
struct DiagGen {
  double D2[81];  // D2[q*n+i] = Dgl[q][i]^2
  double dd[9];   // diag of Dgl
};
static __global__ void k_diag_general(BrickGrid g, GeoMesh gm, PointTab pt, DiagGen dg, i64 n_cells,
                                      double* __restrict__ diag, int* __restrict__ error) {
  __shared__ double nodes[81];
  extern __shared__ double Gs[];  // [n^3][6]
  const int p = g.p, n = p + 1, n3 = n * n * n;
  for (i64 cell = blockIdx.x; cell < n_cells; cell += gridDim.x) {
    __syncthreads();
    cell_nodes_to_smem(gm, cell, nodes);
    __syncthreads();
    for (int q = threadIdx.x; q < n3; q += blockDim.x) {
      const int i = q % n, j = (q / n) % n, k = q / (n * n);
      double J[9], inv[9], g6[6];
      jacobian27(nodes, pt.qv + 3 * i, pt.qd + 3 * i, pt.qv + 3 * j, pt.qd + 3 * j, pt.qv + 3 * k, pt.qd + 3 * k, J);
      const double det = invert3(J, inv);
      if (!(det > 0.0)) *error = 1;
      tensor6(inv, det * (pt.w[k] * pt.w[j] * pt.w[i]), g6);
      for (int c = 0; c < 6; ++c) Gs[q * 6 + c] = g6[c];
    }
    __syncthreads();
    const int cx = (int)(cell % g.cells[0]), cy = (int)((cell / g.cells[0]) % g.cells[1]),
              cz = (int)(cell / ((i64)g.cells[0] * g.cells[1]));
    for (int q = threadIdx.x; q < n3; q += blockDim.x) {
      const int i = q % n, j = (q / n) % n, k = q / (n * n);
      double lap = 0.0;
      for (int t = 0; t < n; ++t) {
        lap += dg.D2[t * n + i] * Gs[((k * n + j) * n + t) * 6 + 0];
        lap += dg.D2[t * n + j] * Gs[((k * n + t) * n + i) * 6 + 1];
        lap += dg.D2[t * n + k] * Gs[((t * n + j) * n + i) * 6 + 2];
      }
      const double* gq = Gs + q * 6;
      lap += 2.0 * (dg.dd[i] * dg.dd[j] * gq[3] + dg.dd[i] * dg.dd[k] * gq[4] + dg.dd[j] * dg.dd[k] * gq[5]);
      atomicAdd(&diag[lattice_to_dev(g, cx * p + i, cy * p + j, cz * p + k)], lap);
    }
  }
}

}  // namespace mfcg
