/*
 * mfcg_b200.h -- C ABI of the B200-native matrix-free CG hot path.
 *
 * The reference (`/root/reference/pkg/src/mfcg`) is pure Python and has no FFI
 * layer; its boundary for this path is the duck-typed operator protocol between
 * `solvers.py` and `operator.py`.  Each entry point below names the reference
 * interface it stands in for (file:line relative to pkg/src/mfcg).  The Python
 * package `paper_2205_08909_b200` binds these symbols with ctypes and is the
 * only caller; see INTEGRATION.md for the stub a maintainer of the reference
 * would add.
 *
 * Conventions
 *   - every function returns an int status (MFCG_OK == 0) and never throws;
 *     `mfcg_last_error()` returns the message of the last failure on the
 *     calling thread.
 *   - all vectors cross this boundary in the CALLER's DoF numbering (the one of
 *     `cell_index_blocks`), as fp64, either in host memory (location 0) or in
 *     device memory of the context's GPU (location 1).  Inside, the library
 *     keeps vectors in its own brick numbering; the
 *     permutation is applied on the device at the boundary.
 *   - integer tables (numbering, constraints) are consumed, never re-derived:
 *     bit-exact numbering is checkable at this boundary.
 */
#ifndef MFCG_B200_H
#define MFCG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFCG_OK            0
#define MFCG_EINVAL        1   /* -> ValueError                          */
#define MFCG_ENOMEM        2   /* -> MemoryError                         */
#define MFCG_ECUDA         3   /* -> RuntimeError                        */
#define MFCG_EBREAKDOWN    4   /* -> SolverBreakdown (solvers.py:36-37)  */
#define MFCG_EUNSUPPORTED  5   /* -> NotImplementedError                 */

/* geometry variants, mesh.py:40-47 */
#define MFCG_GEOM_AFFINE                0
#define MFCG_GEOM_FINAL_TENSOR_LOAD     1
#define MFCG_GEOM_INVERSE_JACOBIAN_LOAD 2
#define MFCG_GEOM_QUADRATIC_COMPUTE     3

/* solver variants, solvers.py:34 (pipelined / sstep are out of scope) */
#define MFCG_CG           0
#define MFCG_PCG          1
#define MFCG_COMBINED_CG  2
#define MFCG_COMBINED_PCG 3

/* breakdown codes returned in mfcg_solve_result.breakdown */
#define MFCG_BRK_NONE 0
#define MFCG_BRK_PAP  1   /* p^T A p <= 0           solvers.py:222-227, 734-742 */
#define MFCG_BRK_RMR  2   /* r^T M^-1 r <= 0        solvers.py:724-727          */
#define MFCG_BRK_BETA 3   /* recurrence beta <= 0   solvers.py:748-756          */

typedef struct mfcg_ctx mfcg_ctx;
typedef struct mfcg_op mfcg_op;

/* One CUDA device, one stream (+ NCCL communicator when slabs are used). */
int mfcg_ctx_create(int device, mfcg_ctx** ctx);
void mfcg_ctx_destroy(mfcg_ctx* ctx);
const char* mfcg_last_error(void);
/* The cudaStream_t all work of this context is enqueued on (for event timing by the caller). */
void* mfcg_ctx_stream(mfcg_ctx* ctx);

/*
 * Operator description == arguments of `MatrixFreeOperator(spec, mesh, handler,
 * plan)` (operator.py:130-176) flattened to plain arrays.
 */
typedef struct mfcg_op_desc {
  int32_t degree;                 /* OperatorSpec.degree                                  */
  int32_t n_q_1d;                 /* OperatorSpec.n_q_1d                                  */
  const double* shape_values;     /* basis.shape_values   [n_q][p+1]  tensor.py:223-239   */
  const double* shape_gradients;  /* basis.shape_gradients[n_q][p+1]                      */
  const double* quad_points;      /* quadrature.points [n_q] on [0,1]                     */
  const double* quad_weights;     /* quadrature.weights[n_q]                              */
  const double* gl_points;        /* (p+1)-point Gauss-Lobatto rule used by               */
  const double* gl_weights;       /*   compute_diagonal (operator.py:384-386)             */
  const double* gl_gradients;     /* its collocation derivative [p+1][p+1]                */
  int32_t cells[3];               /* HexMesh.cells_per_dim                                */
  double extents[3];              /* HexMesh.extents                                      */
  double deformation;             /* HexMesh.deformation (mesh.py:73-80)                  */
  const int32_t* cell_index_blocks; /* DofHandler.cell_index_blocks [n_cells][27]         */
  int64_t n_dofs;                 /* DofHandler.n_dofs                                    */
  const int64_t* constrained;     /* DofHandler.constrained_dofs                          */
  int64_t n_constrained;
  int32_t geometry;               /* MFCG_GEOM_*                                          */
  int32_t precision;              /* 0 = fp64 (reference), 1 = fp32 vectors + operator    */
  int32_t brick[3];               /* cells per thread-block brick; 0 = library default    */
  /* z-slab decomposition; single GPU: slab_cells_z = cells[2], offset 0 */
  int32_t slab_z0;                /* first global cell layer of this slab                 */
  int32_t global_cells_z;         /* cell layers of the whole mesh (0: cells[2]); with    */
                                  /* slabs, `cells` is the slab and `extents` the mesh    */
  int32_t components;             /* OperatorSpec.components: 1 or 3 (0 reads as 1); with 3, */
                                  /* vectors interleave the components of a node             */
                                  /* (dofs.py:229-236), n_dofs = 3 * nodes and `constrained` */
                                  /* lists whole nodes; the diagonal stays one value per node */
} mfcg_op_desc;

int mfcg_op_create(mfcg_ctx* ctx, const mfcg_op_desc* desc, mfcg_op** op);
void mfcg_op_destroy(mfcg_op* op);

typedef struct mfcg_op_info {
  int64_t n_dofs;
  int64_t n_interior;     /* DoFs private to one brick (fused fully on chip)      */
  int64_t n_bricks;
  int32_t brick[3];
  int32_t threads;        /* threads per brick kernel block                       */
  int32_t smem_bytes;     /* dynamic shared memory per block                      */
  int64_t geometry_bytes; /* device bytes held for the geometry variant           */
} mfcg_op_info;
int mfcg_op_get_info(mfcg_op* op, mfcg_op_info* info);

/* perm[user index] = device (brick-numbering) index; length n_dofs. */
int mfcg_op_device_permutation(mfcg_op* op, int32_t* perm_host);

/* dst = A src; replaces MatrixFreeOperator.apply (operator.py:285-292).
 * src/dst: fp64[n_dofs], caller numbering; location 0 host / 1 device.
 * With 3 components the scalar operator acts on each component (operator.py:256-281). */
int mfcg_op_apply(mfcg_op* op, const double* src, double* dst, int location);

/* 1/diag of the GL-collocation operator, constrained entries 1; replaces
 * MatrixFreeOperator.compute_diagonal (operator.py:380-418).
 * inv_diag: fp64[n_dofs / components] (one value per node, operator.py:90).
 * Returns MFCG_EINVAL "operator diagonal is not positive definite" like :416-417. */
int mfcg_op_diagonal(mfcg_op* op, double* inv_diag, int location);

/* The geometry table the device computed for the operator's own quadrature:
 * kind 1 -> final tensor [n_cells][n_q^3][6] (mesh.py:194-201 order xx,yy,zz,xy,xz,yz),
 * kind 2 -> inverse Jacobian [n_cells][n_q^3][9] followed by jxw [n_cells][n_q^3].
 * For parity tests against mesh.precompute_geometry (mesh.py:209-252). */
int mfcg_op_geometry(mfcg_op* op, int kind, double* out_host, int64_t n_doubles);

typedef struct mfcg_solve_args {
  int32_t variant;            /* MFCG_CG ...                                         */
  int32_t location;           /* of b, inv_diag, x: 0 host, 1 device                 */
  const double* b;            /* right-hand side [n_dofs]                            */
  const double* inv_diag;     /* scalar inverse diagonal [n_dofs / components] or NULL */
  double* x;                  /* out: solution [n_dofs]                              */
  double tolerance;           /* SolverConfig.tolerance      solvers.py:41           */
  int32_t max_iterations;     /* SolverConfig.max_iterations                         */
  int32_t fixed_iterations;   /* SolverConfig.fixed_iterations, -1 = None            */
  int32_t force_x_updates;    /* SolverConfig.force_x_updates                        */
  int32_t fused;              /* combined_*: 1 = fused brick kernel, 0 = pre/apply/post kernels */
  int32_t time_kernels;       /* 1 = CUDA-event time the operator kernel per launch   */
  double* history;            /* out (host): [limit][4] = alpha, beta, gamma, residual */
} mfcg_solve_args;

typedef struct mfcg_solve_result {
  int32_t iterations;
  int32_t converged;
  int32_t matvecs;
  int32_t breakdown;          /* MFCG_BRK_*                                          */
  int32_t breakdown_iteration;
  double breakdown_value;
  double residual;            /* final relative residual                             */
  double bnorm;
  double solve_ms;            /* device time of the whole solve (CUDA events)        */
  double operator_ms;         /* device time inside the operator kernel(s), if timed */
  int64_t kernel_launches;    /* kernels of this library launched by the solve       */
  int64_t operator_launches;
} mfcg_solve_result;

/* Replaces solve()/solve_cg/solve_pcg/solve_combined_cg/solve_combined_pcg
 * (solvers.py:183, 257, 795, 805, 816-834).  x0 = 0.  Zero rhs -> iterations 0. */
int mfcg_solve(mfcg_op* op, const mfcg_solve_args* args, mfcg_solve_result* result);

/* Slab exchange hooks: the library calls NCCL itself once the
 * communicator is set.  unique_id is the 128-byte ncclUniqueId from rank 0. */
int mfcg_comm_unique_id(void* unique_id_128);
int mfcg_ctx_init_comm(mfcg_ctx* ctx, const void* unique_id_128, int rank, int n_ranks);

/* Slab groups: `ops` are adjacent z-slabs held by this process (bottom to top, one context).
 * Neighbours inside the group exchange the shared lattice plane by device-to-device copies,
 * the slabs below / above the group by ncclSend/ncclRecv with ranks rank-1 / rank+1; the seven
 * sums of a merged iteration are reduced over the group and with one ncclAllReduce over ranks.
 * One process per GPU uses n_ops == 1.  (No reference counterpart.) */
int mfcg_apply_group(mfcg_op** ops, int n_ops, const double* const* src, double* const* dst, int location);
int mfcg_diagonal_group(mfcg_op** ops, int n_ops, double* const* inv_diag, int location);
int mfcg_solve_group(mfcg_op** ops, int n_ops, const mfcg_solve_args* args, mfcg_solve_result* results);

#ifdef __cplusplus
}
#endif
#endif /* MFCG_B200_H */
