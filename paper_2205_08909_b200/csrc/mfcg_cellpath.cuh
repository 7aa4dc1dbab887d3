// mfcg_cellpath.cuh -- cell-by-cell Laplace apply for curved meshes with n_q_1d > p + 1.
//
// The reference accepts any n_q_1d >= p + 1 (operator.py:69-70) and its BP3 / BP4 problems use p + 2 points on
// the deformed mesh (bench.py:62-63).  The brick kernels hold (p+1)^3 tiles and cover n_q = p + 1 (every
// BASELINE configuration); this kernel covers the rest the way the reference does it: per cell gather
// (constrained entries -> 0), the nine sweeps of evaluate_gradients with the rectangular S and D
// (tensor.py:335-347), flux = G grad (operator.py:271-274), the nine transposed sweeps of integrate_gradients
// (tensor.py:357-370), scatter-add (operator.py:338-353).  One block per cell, everything in shared memory,
// global atomics for the scatter: a correctness path (BP3 / BP4 as the reference defines them), not a tuned one.
#pragma once
#include "mfcg_kernels.cuh"

namespace mfcg {

struct CellTables {
  int n, nq;            // p + 1 and n_q_1d (<= 10)
  double S[10 * 9];     // S[q * n + i] = phi_i(x_q)
  double D[10 * 9];     // D[q * n + i] = phi_i'(x_q)
};

template <typename T>
__global__ void __launch_bounds__(128)
k_cell_general(BrickGrid g, CellTables ct, GeomAccess geo, PointTab pt, i64 n_cells, const T* __restrict__ src,
               T* __restrict__ dst) {
  extern __shared__ __align__(16) unsigned char cell_smem[];
  const int n = ct.n, nq = ct.nq, n3 = n * n * n, q3n = nq * nq * nq;
  T* buf[6];
  for (int b = 0; b < 6; ++b) buf[b] = reinterpret_cast<T*>(cell_smem) + (size_t)b * q3n;
  int* idx = reinterpret_cast<int*>(reinterpret_cast<T*>(cell_smem) + (size_t)6 * q3n);  // device index, -1 - index if constrained
  __shared__ T Ss[90], Ds[90];
  __shared__ double nodes[81];
  for (int t = threadIdx.x; t < nq * n; t += blockDim.x) { Ss[t] = (T)ct.S[t]; Ds[t] = (T)ct.D[t]; }
  const int p = g.p;
  for (i64 cell = blockIdx.x; cell < n_cells; cell += gridDim.x) {
    __syncthreads();
    const int cx = (int)(cell % g.cells[0]), cy = (int)((cell / g.cells[0]) % g.cells[1]),
              cz = (int)(cell / ((i64)g.cells[0] * g.cells[1]));
    T* U = buf[5];
    for (int t = threadIdx.x; t < n3; t += blockDim.x) {
      const int i = t % n, j = (t / n) % n, k = t / (n * n);
      const i64 d = lattice_to_dev(g, cx * p + i, cy * p + j, cz * p + k);
      const bool con = d >= g.n_int && (g.mask[d - g.n_int] & 1);
      idx[t] = con ? -1 - (int)d : (int)d;
      U[t] = con ? (T)0 : src[d];                        // operator.py:341-342
    }
    if (geo.kind == 3)
      for (int t = threadIdx.x; t < 81; t += blockDim.x) nodes[t] = reinterpret_cast<const double*>(geo.data)[cell * 81 + t];
    __syncthreads();
    // x: A = Sx u, B = Dx u                              (n, n, nq)
    T *A = buf[0], *B = buf[1];
    for (int t = threadIdx.x; t < n * n * nq; t += blockDim.x) {
      const int q = t % nq, line = t / nq;
      T a = 0, b = 0;
      for (int i = 0; i < n; ++i) { const T u = U[line * n + i]; a += Ss[q * n + i] * u; b += Ds[q * n + i] * u; }
      A[t] = a; B[t] = b;
    }
    __syncthreads();
    // y: AA = Sy A, AD = Dy A, BA = Sy B                  (n, nq, nq)
    T *AA = buf[2], *AD = buf[3], *BA = buf[4];
    for (int t = threadIdx.x; t < n * nq * nq; t += blockDim.x) {
      const int q1 = t % nq, q2 = (t / nq) % nq, k = t / (nq * nq);
      T aa = 0, ad = 0, ba = 0;
      for (int j = 0; j < n; ++j) {
        const T a = A[(k * n + j) * nq + q1], b = B[(k * n + j) * nq + q1];
        aa += Ss[q2 * n + j] * a; ad += Ds[q2 * n + j] * a; ba += Ss[q2 * n + j] * b;
      }
      AA[t] = aa; AD[t] = ad; BA[t] = ba;
    }
    __syncthreads();
    // z and the flux at every quadrature point            (nq, nq, nq)
    T *FX = buf[0], *FY = buf[1], *FZ = buf[5];
    for (int t = threadIdx.x; t < q3n; t += blockDim.x) {
      const int q1 = t % nq, q2 = (t / nq) % nq, q3 = t / (nq * nq);
      T gx = 0, gy = 0, gz = 0;
      for (int k = 0; k < n; ++k) {
        const int o = (k * nq + q2) * nq + q1;
        gx += Ss[q3 * n + k] * BA[o]; gy += Ss[q3 * n + k] * AD[o]; gz += Ds[q3 * n + k] * AA[o];
      }
      T G6[6];
      if (geo.kind == 1) {
        const T* gp = reinterpret_cast<const T*>(geo.data) + ((i64)cell * q3n + t) * 6;
        for (int c = 0; c < 6; ++c) G6[c] = gp[c];
      } else {
        double inv[9], jxw, g6d[6];
        if (geo.kind == 2) {
          const T* ip = reinterpret_cast<const T*>(geo.data) + ((i64)cell * q3n + t) * 9;
          for (int c = 0; c < 9; ++c) inv[c] = (double)ip[c];
          jxw = (double)reinterpret_cast<const T*>(geo.jxw)[(i64)cell * q3n + t];
        } else {
          double J[9];
          jacobian27(nodes, pt.qv + 3 * q1, pt.qd + 3 * q1, pt.qv + 3 * q2, pt.qd + 3 * q2, pt.qv + 3 * q3, pt.qd + 3 * q3, J);
          const double det = invert3(J, inv);
          jxw = det * (pt.w[q3] * pt.w[q2] * pt.w[q1]);
        }
        tensor6(inv, jxw, g6d);
        for (int c = 0; c < 6; ++c) G6[c] = (T)g6d[c];
      }
      FX[t] = G6[0] * gx + G6[3] * gy + G6[4] * gz;        // operator.py:271-274
      FY[t] = G6[3] * gx + G6[1] * gy + G6[5] * gz;
      FZ[t] = G6[4] * gx + G6[5] * gy + G6[2] * gz;
    }
    __syncthreads();
    // z^T: P1 = Sz^T fx, P2 = Sz^T fy, P3 = Dz^T fz       (n, nq, nq)
    T *P1 = buf[2], *P2 = buf[3], *P3 = buf[4];
    for (int t = threadIdx.x; t < n * nq * nq; t += blockDim.x) {
      const int q1 = t % nq, q2 = (t / nq) % nq, k = t / (nq * nq);
      T a = 0, b = 0, c = 0;
      for (int q3 = 0; q3 < nq; ++q3) {
        const int o = (q3 * nq + q2) * nq + q1;
        a += Ss[q3 * n + k] * FX[o]; b += Ss[q3 * n + k] * FY[o]; c += Ds[q3 * n + k] * FZ[o];
      }
      P1[t] = a; P2[t] = b; P3[t] = c;
    }
    __syncthreads();
    // y^T: Q1 = Sy^T P1 (x-derivative part), Q2 = Dy^T P2 + Sy^T P3   (n, n, nq)
    T *Q1 = buf[0], *Q2 = buf[1];
    for (int t = threadIdx.x; t < n * n * nq; t += blockDim.x) {
      const int q1 = t % nq, j = (t / nq) % n, k = t / (nq * n);
      T a = 0, b = 0;
      for (int q2 = 0; q2 < nq; ++q2) {
        const int o = (k * nq + q2) * nq + q1;
        a += Ss[q2 * n + j] * P1[o];
        b += Ds[q2 * n + j] * P2[o] + Ss[q2 * n + j] * P3[o];
      }
      Q1[t] = a; Q2[t] = b;
    }
    __syncthreads();
    // x^T and scatter-add; constrained rows are dropped (operator.py:348-353)
    for (int t = threadIdx.x; t < n3; t += blockDim.x) {
      const int i = t % n, line = t / n;
      T a = 0;
      for (int q1 = 0; q1 < nq; ++q1) a += Ds[q1 * n + i] * Q1[line * nq + q1] + Ss[q1 * n + i] * Q2[line * nq + q1];
      if (idx[t] >= 0) atomicAdd(&dst[idx[t]], a);
    }
  }
}

// dst[c] = src[c] on constrained DoFs after the scatter (operator.py:359-360) is k_surface_fix.

}  // namespace mfcg
