// mfcg_brick2.cuh -- the merged-CG iteration on affine meshes as a persistent, TMA-fed kernel.
//
// Same mathematics and the same brick numbering as k_brick<P, T, 1, 0> (mfcg_kernels.cuh; reference
// semantics solvers.py:660-704 + operator.py:338-360), re-organised around what bounded that kernel on
// B200 (profiles/r01_final_ncu_brick.txt: L1 data pipe 76 % busy, long_scoreboard the top stall):
//
//   * one persistent block per SM walks a list of bricks; three roles, each with its own pace:
//       producer (1 elected lane)  streams the contiguous interior runs of r, p, v (, x) plane by plane
//                                  with cp.async.bulk (SASS UBLKCP) into shared memory, and writes r', p'
//                                  (, x') back with bulk stores -- no interior value crosses a register on
//                                  its way in or out;
//       update warps (96 threads)  do the "pre" update (solvers.py:660-690) in place in the staged planes,
//                                  copy p' into the lattice-plane ring, take r.r and r.Mr, and fetch the
//                                  brick-boundary values of p;
//       math warps (128 threads)   one thread per (cell, z-plane): the plane's (p+1)^2 values go to
//                                  registers, the x and y sweeps run there, only the z sweep goes through
//                                  shared memory (6 instead of 10 shared-memory accesses per tile entry);
//                                  then the deterministic gather, v stores, and the five sums that need v
//                                  -- taken on r' and p' that never left the SM (no re-read through L2).
//   * r' stays staged for the layers in flight (NRL layers), p, v, x pass through NT transient plane slots.
//
// Hand-over: mbarriers with running phase counters (they are never re-initialised between bricks, so the
// producer and the update warps run ahead into the next brick while the math warps finish the current one).
#pragma once
#include <type_traits>

#include "mfcg_kernels.cuh"

namespace mfcg {

// ---- bulk-copy (TMA) helpers
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, unsigned src_smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int NPEND> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NPEND) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy writes to shared memory become visible to the async proxy (bulk stores)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void pin_value(double& v) { asm volatile("" : "+d"(v)); }
__device__ __forceinline__ void pin_value(float& v) { asm volatile("" : "+f"(v)); }
__device__ __forceinline__ void pin_value(unsigned& v) { asm volatile("" : "+r"(v)); }
template <class U> __device__ __forceinline__ void pin_value(U*& v) { asm volatile("" : "+l"(v)); }
// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  unsigned pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
template <int ID, int COUNT> __device__ __forceinline__ void named_barrier() {
  asm volatile("barrier.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");  // non-aligned: lanes of a warp may arrive from different places
}

template <int ID, int COUNT> __device__ __forceinline__ void named_arrive() {
  asm volatile("barrier.arrive %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}

#ifndef MFCG_B2_SKIP
#define MFCG_B2_SKIP 0  // timing experiments only (wrong results): 1 no global stores in the update, 2 no ring
                        // stores, 4 no update at all, 8 no gather, 16 no z sweep, 32 no plane sweeps
#endif
#ifndef MFCG_B2_NT
#define MFCG_B2_NT 4   // transient plane slots (p, v, x)
#endif
#ifndef MFCG_B2_RLAYERS
#define MFCG_B2_RLAYERS 3  // layers of lattice planes in the ring: the update runs RLAYERS - 1 layers ahead of the gather
#endif
#ifndef MFCG_B2_UNR
#define MFCG_B2_UNR 2
#endif
#ifndef MFCG_B2_PMIN
#define MFCG_B2_PMIN 4  // lowest degree that runs in the persistent kernel
#endif
#ifndef MFCG_B2_UNIFORM_PRODUCER
#define MFCG_B2_UNIFORM_PRODUCER 1  // producer warp runs converged, an elected lane issues the bulk copies
#endif
#ifndef MFCG_B2_REGTAB
#define MFCG_B2_REGTAB 1  // update warps keep their granules' table entries in registers (fp64, shared planes)
#endif
#ifndef MFCG_B2_LOOPUNR
#define MFCG_B2_LOOPUNR 1  // unroll of the update loop over granule pairs
#endif
#ifndef MFCG_B2_UNRX
#define MFCG_B2_UNRX 1
#endif
#ifndef MFCG_B2_NRL
#define MFCG_B2_NRL 4  // layers of r' staged on chip (3 ring layers, 4 slots, 4 staged layers: best of the combinations
                       // that fit 227 KB, profiles/r02_notes.md)
#endif

#ifdef MFCG_TIMING
#define B2_TIC(v) long long v = clock64()
#define B2_TOC(v, slot) do { long long n__ = clock64(); tacc[slot] += (unsigned long long)(n__ - v); v = n__; } while (0)
#else
#define B2_TIC(v)
#define B2_TOC(v, slot)
#endif

template <int P> struct Brick2Enabled {
  // needs a multiple of 16 cells per layer (cell-minor mapping) and N^2 * 2 values of a plane in registers.
  // Measured at ~5e7 DoFs (profiles/r02_sweeps.txt): p = 5 +5 %, p = 4 +1 %, but p = 3 / 2 -13 / -10 % against
  // the first-generation kernel (many small planes per layer: the per-plane hand-over costs more than the
  // register-resident sweeps save), so the low degrees stay there.
  static constexpr bool value = (P >= MFCG_B2_PMIN && P <= 5) && (Cfg<P, 0>::BX * Cfg<P, 0>::BY) % 16 == 0;
};

template <int P, typename T> struct Geo2 {
  static constexpr int N = P + 1, BX = Cfg<P, 0>::BX, BY = Cfg<P, 0>::BY, NCELL = BX * BY;
  static constexpr int RS = N, PSTR = N * N, TILE = Geo<P, 0>::TILE;
  static constexpr int WX = P * BX + 1;                       // lattice row pitch
  static constexpr int LXM = P * BX - 1, LYM = P * BY - 1, NINT2D = LXM * LYM;
  static constexpr int FP_MAX = (P * BX + 1) * (P * BY + 1);
  // ring of lattice planes: three consecutive layers, also across brick boundaries (3 x (P+1) planes): the
  // update warps may run two layers ahead of the gather
  static constexpr int RLAYERS = MFCG_B2_RLAYERS, RB = RLAYERS * (P + 1);
  static constexpr int PER16 = 16 / (int)sizeof(T);
  static constexpr int NT = MFCG_B2_NT, NRL = MFCG_B2_NRL;
  // 16 warps: 0-2 plane sweeps in registers (NS1), 3 producer, 4-11 z sweep + gather (NLM), 12-15 update (NUPD).
  // (7 + 5 warps for gather / update measured 5 % slower at 116^3, profiles/r02_notes.md)
  static constexpr int NS1 = 96, NLM = 256, NUPD = 128, THREADS = 512;
  static constexpr int REG_S1 = 232, REG_LIGHT = 88, REG_UPD = 104;  // setmaxnreg per warpgroup: 128 * (232 + 2 * 88 + 104) == 512 * 128
  // Rows of cell row cy are shifted by SK * cy so that the 16 (fp64) / 32 (fp32) lanes of a shared-memory
  // wavefront -- the same plane entry of consecutive cells -- fall into different banks.
  static constexpr int bank_conflicts(int sk) {
    const int lanes = sizeof(T) == 8 ? 16 : 32;
    const int nb = lanes;  // banks in units of sizeof(T)
    int worst = 0;
    for (int b = 0; b < nb; ++b) {
      int cnt = 0;
      for (int c = 0; c < lanes && c < NCELL; ++c) {
        const int cy = c / BX, cx = c - cy * BX;
        if ((cy * (P * WX + sk) + cx * P) % nb == b) ++cnt;
      }
      if (cnt > worst) worst = cnt;
    }
    return worst;
  }
  static constexpr int skew() {
    int best = 0, bw = bank_conflicts(0);
    for (int s = 1; s < 32; ++s) {
      const int w = bank_conflicts(s);
      if (w < bw) { bw = w; best = s; }
    }
    return best;
  }
  static constexpr int SK = skew();
  static constexpr int PLANE = WX * (P * BY + 1) + SK * BY;   // last lattice row carries the shift SK * BY
  static constexpr int PLB = (((NINT2D + 2 * PER16) * (int)sizeof(T) + 127) / 128 * 128) / (int)sizeof(T);  // staged plane, elements
  static_assert(NINT2D <= 32 * NUPD && FP_MAX - NINT2D <= NUPD, "one update thread per brick-boundary position of a plane");
  static_assert(PLANE < 1024 && NINT2D < 4096 && P * P < 64 && NCELL * TILE < 16384, "packed table fields");

  static constexpr size_t al(size_t x) { return (x + 127) & ~(size_t)127; }
  static constexpr size_t OFF_RING = 2048;
  static constexpr size_t OFF_CARRY = al(OFF_RING + sizeof(T) * RB * PLANE);
  static constexpr size_t OFF_A = al(OFF_CARRY + sizeof(T) * PLANE);
  static constexpr size_t OFF_B = al(OFF_A + sizeof(T) * NCELL * TILE);
  static constexpr size_t OFF_R = al(OFF_B + sizeof(T) * NCELL * TILE);
  static constexpr size_t OFF_T = al(OFF_R + sizeof(T) * NRL * P * PLB);
  static constexpr size_t OFF_DTAB = al(OFF_T + sizeof(T) * NT * 3 * PLB);
  static constexpr size_t OFF_GTAB = al(OFF_DTAB + sizeof(T) * P * P * P);
  static constexpr size_t OFF_ITAB = al(OFF_GTAB + 8 * (size_t)FP_MAX);
  static constexpr size_t SMEM = al(OFF_ITAB + 2 * (size_t)NINT2D);
  static_assert(SMEM <= 232448 - 1024, "shared memory of the persistent brick kernel");
};

struct Hdr2 {
  i64 st27[3][28];                       // 27 entity starts of the current brick, one copy per role
  unsigned long long tfull[8], tupd[8];  // transient slot loaded / updated
  unsigned long long lfull[4], ldone[4]; // layer ready for the math warps / gather of a layer finished
  double lsum[4][8][2];                  // r.r and r.Mr of a layer, per update warp
  double bsum[2];                        // their running sums over the brick
  double red[8][8];
};
static_assert(sizeof(Hdr2) <= 2048, "header");

template <int P, typename T>
__global__ void __launch_bounds__(512, 1)
k_brick2(BrickGrid g, SepTables<T, P + 1> tab, int diag_mode, T* __restrict__ Pv, T* __restrict__ V,
         T* __restrict__ R, T* __restrict__ X, const SolveState* __restrict__ st, double* __restrict__ partials,
         int brick_first, int brick_count) {
  using G2 = Geo2<P, T>;
  constexpr int N = P + 1, RS = G2::RS, PSTR = G2::PSTR, TILE = G2::TILE, WX = G2::WX, SK = G2::SK,
                PLANE = G2::PLANE, NCELL = G2::NCELL, RB = G2::RB, PER16 = G2::PER16, PLB = G2::PLB,
                NT = G2::NT, NRL = G2::NRL, NS1 = G2::NS1, NLM = G2::NLM, NUPD = G2::NUPD, HE = EOShape<N>::HE,
                NTHR = G2::THREADS, T_PROD = NS1, T_LM = 128, T_UPD = 128 + NLM;
  static_assert(T_UPD + NUPD == NTHR && T_UPD % 128 == 0, "thread map: roles with different register budgets fill whole warpgroups");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Hdr2& H = *reinterpret_cast<Hdr2*>(smem_raw);
  T* const ring = reinterpret_cast<T*>(smem_raw + G2::OFF_RING);
  T* const carry = reinterpret_cast<T*>(smem_raw + G2::OFF_CARRY);
  T* const A = reinterpret_cast<T*>(smem_raw + G2::OFF_A);
  T* const Bs = reinterpret_cast<T*>(smem_raw + G2::OFF_B);
  T* const Rbuf = reinterpret_cast<T*>(smem_raw + G2::OFF_R);
  T* const Tbuf = reinterpret_cast<T*>(smem_raw + G2::OFF_T);
  T* const dtab = reinterpret_cast<T*>(smem_raw + G2::OFF_DTAB);
  uint2* const gtab = reinterpret_cast<uint2*>(smem_raw + G2::OFF_GTAB);
  unsigned short* const itab = reinterpret_cast<unsigned short*>(smem_raw + G2::OFF_ITAB);

  const int tid = threadIdx.x;
  if (!st->active) return;
  const T am1 = (T)st->am1, bm1 = (T)st->bm1, xc1 = (T)st->xc1, xc2 = (T)st->xc2;
  const int xmode = st->xmode;

  if (tid == 0) {
    for (int i = 0; i < NT; ++i) { mbar_init(&H.tfull[i], 1); mbar_init(&H.tupd[i], NUPD); }
    for (int i = 0; i < 4; ++i) mbar_init(&H.lfull[i], NUPD);
    for (int i = 0; i < 4; ++i) mbar_init(&H.ldone[i], NLM);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < P * P * P; i += NTHR)
    dtab[i] = diag_mode == 1 ? diag_inverse_onfly<T, N>(tab, i % P, (i / P) % P, i / (P * P)) : (T)1;

  // lattice point (i, j) of a layer -> offset inside a ring plane
  auto ring_off = [](int i, int j) { return j * WX + i + SK * (j / P); };

  // Tables of a brick shape (bcx x bcy cells per layer), shared by all roles.
  //  gtab: per lattice point of a layer, sorted (points strictly inside a cell, brick-boundary points in
  //        perimeter order, other cell-boundary points):
  //        x: tile offset [0,14) | which of the four cells around exist [14,18) | brick-boundary flag 18 |
  //           macro entity [19,23) | 1/diag class in the plane [23,30)
  //        y: ring offset [0,10) | offset inside the macro entity [10,22) | plane-stride selector [22,24)
  //  itab: per interior point of a plane: ring offset | 1/diag class << 10
  auto build_tables = [&](int bcx, int bcy) {
    const int Lx = P * bcx, Ly = P * bcy, fw_ = Lx + 1;
    const int rowc = bcx * (P - 1), n_in = rowc * bcy * (P - 1), nper = 2 * fw_ + 2 * (Ly - 1);
    for (int rem = tid; rem < fw_ * (Ly + 1); rem += NTHR) {
      const int j = rem / fw_, i = rem - j * fw_;
      const int cx1 = i / P, ix1 = i - cx1 * P, cy1 = j / P, iy1 = j - cy1 * P;
      const int rows_before = cy1 * (P - 1) + (iy1 == 0 ? 0 : iy1 - 1);
      const int in_row_before = cx1 * (P - 1) + (ix1 == 0 ? 0 : ix1 - 1);
      const int before = rows_before * rowc + (iy1 != 0 ? in_row_before : 0);
      int pos;
      if (ix1 != 0 && iy1 != 0) pos = before;
      else if (j == 0) pos = n_in + i;
      else if (j == Ly) pos = n_in + fw_ + i;
      else if (i == 0 || i == Lx) pos = n_in + 2 * fw_ + 2 * (j - 1) + (i == Lx ? 1 : 0);
      else pos = n_in + nper + (rem - before - (fw_ + 2 * (j - 1) + 1));
      MFCG_CHECK(pos >= 0 && pos < G2::FP_MAX);
      const int ex = i == 0 ? 0 : (i == Lx ? 2 : 1), ey = j == 0 ? 0 : (j == Ly ? 2 : 1);
      const int ox = ex == 1 ? i - 1 : 0, oy = ey == 1 ? j - 1 : 0;
      const int lx = ex == 1 ? Lx - 1 : 1;
      const unsigned base = (unsigned)((cy1 * bcx + cx1) * TILE + iy1 * RS + ix1);
      const unsigned v11 = cx1 < bcx && cy1 < bcy, v10 = ix1 == 0 && cx1 > 0 && cy1 < bcy,
                     v01 = iy1 == 0 && cy1 > 0 && cx1 < bcx, v00 = ix1 == 0 && iy1 == 0 && cx1 > 0 && cy1 > 0;
      const unsigned edge = (ex != 1) || (ey != 1);
      const unsigned sel = (ex == 1 ? 1u : 0u) | (ey == 1 ? 2u : 0u);
      uint2 d;
      d.x = base | (v11 << 14) | (v10 << 15) | (v01 << 16) | (v00 << 17) | (edge << 18) |
            ((unsigned)(ex + 3 * ey) << 19) | ((unsigned)(iy1 * P + ix1) << 23);
      d.y = (unsigned)ring_off(i, j) | ((unsigned)(ox + lx * oy) << 10) | (sel << 22);
      gtab[pos] = d;
    }
    const int lxm = Lx - 1, n2d = (Lx - 1) * (Ly - 1);
    for (int e = tid; e < n2d; e += NTHR) {
      const int jm = e / lxm, im = e - jm * lxm;
      itab[e] = (unsigned short)(ring_off(im + 1, jm + 1) | ((((jm + 1) % P) * P + (im + 1) % P) << 10));
    }
  };
  __syncthreads();

  const i64 n_int = g.n_int;
  (void)n_int;

  // gather group: the sums that need v (p.v, r.v, v.v, r.Mv, v.Mv) stay in registers over a brick; the update
  // warps hand over r.r and r.Mr with the brick's last layer
  if (tid == 0) { H.bsum[0] = 0.0; H.bsum[1] = 0.0; }  // running r.r, r.Mr of the brick

  // One brick loop per role, each entirely inside its own branch (ptxas allocates registers per
  // setmaxnreg region only when the regions do not re-merge).
  auto run_role = [&](auto role_c) {
  constexpr int ROLE = decltype(role_c)::value;  // 0 plane sweeps, 3 z sweep + gather, 1 producer warp, 2 update warps
  int cur_bcx = -1, cur_bcy = -1;
  int g_base = 0, q_base = 0;  // running layer / plane counters of this block (the barrier phases follow them)
  int kb_base = 0;             // running lattice-plane counter: ring slot of plane K of a brick = (kb_base + K) % RB
#ifdef MFCG_TIMING
  unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0}, tacc6 = 0;
#endif
  for (int bi = blockIdx.x; bi < brick_count; bi += gridDim.x) {
    int b = brick_first + bi;  // a range may wrap around the end of the brick list (top then bottom brick layer of a slab)
    if (b >= g.mb[0] * g.mb[1] * g.mb[2]) b -= g.mb[0] * g.mb[1] * g.mb[2];
    const int mx = b % g.mb[0];
    const int my = (b / g.mb[0]) % g.mb[1];
    const int mz = b / (g.mb[0] * g.mb[1]);
    const int bcx = brick_cells(g, 0, mx), bcy = brick_cells(g, 1, my), bcz = brick_cells(g, 2, mz);
    const int Lx = P * bcx, Ly = P * bcy, Lz = P * bcz;
    const int nint2d = (Lx - 1) * (Ly - 1);
    const int nplanes = nint2d > 0 ? Lz - 1 : 0;
    const int fw = Lx + 1, fp = fw * (Ly + 1);
    if (bcx != cur_bcx || bcy != cur_bcy) {  // every role is between two bricks here
      // non-aligned barrier: the roles arrive from different code, possibly with diverged warps (the aligned
      // bar.sync of __syncthreads() hung here within a few hundred launches on ragged brick grids)
      named_barrier<5, NTHR>();
      build_tables(bcx, bcy);
      named_barrier<5, NTHR>();
      cur_bcx = bcx;
      cur_bcy = bcy;
    }
    auto entity = [&](int t) {
      const int ex = t % 3, ey = (t / 3) % 3, ez = t / 9;
      return g.ent_start[((i64)(2 * mz + ez) * (2 * g.mb[1] + 1) + (2 * my + ey)) * (2 * g.mb[0] + 1) + 2 * mx + ex];
    };

    if constexpr (ROLE == 1) {
      // ================================ producer ================================
#if MFCG_B2_UNIFORM_PRODUCER
      // The whole warp walks the planes with warp-uniform values; one elected lane issues.  (With a single active
      // lane the compiler wraps every bulk copy into an election loop with five register-to-uniform moves.)
      if (nplanes > 0) {
        const i64 st_int = __shfl_sync(0xffffffffu, entity(13), 0);
        for (int K = 1; K <= nplanes; ++K) {
          const int q = q_base + K - 1, slot = q % NT;
          B2_TIC(tp);
          const int gf = g_base + K / P;  // layer whose gather finishes the plane
          const i64 e0 = st_int + (i64)(K - 1) * nint2d;
          const i64 a0 = e0 & ~(i64)(PER16 - 1);
          const int off = (int)(e0 - a0);
          const int len = (off + nint2d + PER16 - 1) & ~(PER16 - 1);
          const unsigned bytes = (unsigned)(len * sizeof(T));
          MFCG_CHECK(len <= PLB && a0 >= 0 && a0 + len <= g.n_dofs + 32 / (int)sizeof(T));
          T* Rb = Rbuf + ((gf % NRL) * P + K % P) * PLB;
          T* Pb = Tbuf + (slot * 3 + 0) * PLB;
          T* Vb = Tbuf + (slot * 3 + 1) * PLB;
          T* Xb = Tbuf + (slot * 3 + 2) * PLB;
          const unsigned tx = bytes * (xmode ? 4u : 3u);
          B2_TOC(tp, 2);
          if (q >= NT) mbar_wait(&H.tupd[slot], ((q - NT) / NT) & 1);  // the slot's previous plane has been read
          B2_TOC(tp, 0);
          if ((K % P == 0 || K == 1) && gf >= NRL) mbar_wait(&H.ldone[(gf - NRL) & 3], ((gf - NRL) >> 2) & 1);
          B2_TOC(tp, 1);
          if (elect_one()) {
            mbar_expect_tx(&H.tfull[slot], tx);
            bulk_g2s(Rb, R + a0, bytes, &H.tfull[slot]);
            bulk_g2s(Pb, Pv + a0, bytes, &H.tfull[slot]);
            bulk_g2s(Vb, V + a0, bytes, &H.tfull[slot]);
            if (xmode) bulk_g2s(Xb, X + a0, bytes, &H.tfull[slot]);
          }
          __syncwarp();
          B2_TOC(tp, 2);
        }
      }
#else
      if ((tid & 31) == 0 && nplanes > 0) {
        const i64 st_int = entity(13);
        for (int K = 1; K <= nplanes; ++K) {
          const int q = q_base + K - 1, slot = q % NT;
          B2_TIC(tp);
          const int gf = g_base + K / P;  // layer whose gather finishes the plane
          const i64 e0 = st_int + (i64)(K - 1) * nint2d;
          const i64 a0 = e0 & ~(i64)(PER16 - 1);
          const int off = (int)(e0 - a0);
          const int len = (off + nint2d + PER16 - 1) & ~(PER16 - 1);
          const unsigned bytes = (unsigned)(len * sizeof(T));
          MFCG_CHECK(len <= PLB && a0 >= 0 && a0 + len <= g.n_dofs + 32 / (int)sizeof(T));
          T* Rb = Rbuf + ((gf % NRL) * P + K % P) * PLB;
          T* Pb = Tbuf + (slot * 3 + 0) * PLB;
          T* Vb = Tbuf + (slot * 3 + 1) * PLB;
          T* Xb = Tbuf + (slot * 3 + 2) * PLB;
          const T* Rs = R + a0; const T* Ps = Pv + a0; const T* Vs = V + a0; const T* Xs = X + a0;
          const unsigned tx = bytes * (xmode ? 4u : 3u);
          pin_value(Rb); pin_value(Pb); pin_value(Vb); pin_value(Xb);
          pin_value(Rs); pin_value(Ps); pin_value(Vs); pin_value(Xs);  // addresses are ready before the waits
          B2_TOC(tp, 2);
          if (q >= NT) mbar_wait(&H.tupd[slot], ((q - NT) / NT) & 1);  // the slot's previous plane has been read
          B2_TOC(tp, 0);
          if ((K % P == 0 || K == 1) && gf >= NRL) mbar_wait(&H.ldone[(gf - NRL) & 3], ((gf - NRL) >> 2) & 1);
          B2_TOC(tp, 1);
          mbar_expect_tx(&H.tfull[slot], tx);
          bulk_g2s(Rb, Rs, bytes, &H.tfull[slot]);
          bulk_g2s(Pb, Ps, bytes, &H.tfull[slot]);
          bulk_g2s(Vb, Vs, bytes, &H.tfull[slot]);
          if (xmode) bulk_g2s(Xb, Xs, bytes, &H.tfull[slot]);
          B2_TOC(tp, 2);
        }
      }
#endif
      __syncwarp();
    } else if constexpr (ROLE == 2) {
      // ================================ update warps ================================
      const int ut = tid - T_UPD, uw = ut >> 5;
      i64* s27 = H.st27[2];
      named_barrier<2, NUPD>();
      if (ut < 27) s27[ut] = entity(ut);
      named_barrier<2, NUPD>();
      const i64 st_int = s27[13];
      double ls0 = 0.0, ls4 = 0.0;  // r.r and r.Mr of this thread over the brick
      // A thread meets the same (at most two) granules of every plane of the brick, shifted by the plane's
      // alignment `off`: their ring offsets and 1/diag classes (itab) stay in registers, so the plane loop has
      // no dependent table load in front of the 1/diag lookup.  tcache[off][round] = entries of the two elements.
      constexpr bool CACHED = MFCG_B2_REGTAB && PER16 == 2 &&
                              ((P * G2::BX - 1) * (P * G2::BY - 1) + 2) / 2 + 1 <= 2 * NUPD;
      unsigned tcache[2][2] = {{0u, 0u}, {0u, 0u}};
      if (CACHED) {
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int e = (par + ut + c * NUPD) * 2 - par;
            const unsigned lo = e < nint2d ? itab[e] : 0u, hi = e + 1 < nint2d ? itab[e + 1] : 0u;
            tcache[par][c] = lo | (hi << 16);
          }
      }
      for (int L = 0; L < bcz; ++L) {
        const int gl = g_base + L;
        B2_TIC(tu);
        // the ring planes this layer overwrites were last read by the gather three layers back
        if (gl >= G2::RLAYERS) mbar_wait(&H.ldone[(gl - G2::RLAYERS) & 3], ((gl - G2::RLAYERS) >> 2) & 1);
        B2_TOC(tu, 0);
        // (the brick-boundary values of the layer's planes are fetched by the plane-sweep warps)
        // (a) interior planes: pre update in place in the staged planes (solvers.py:660-690)
        const int Kfirst = L == 0 ? 1 : L * P + 1;
        const int Klast = L * P + P < Lz - 1 ? L * P + P : Lz - 1;
        if (nint2d > 0)
          for (int K = Kfirst; K <= Klast; ++K) {
            const int q = q_base + K - 1, slot = q % NT;
            const int gf = g_base + K / P;
            T* Rb = Rbuf + ((gf % NRL) * P + K % P) * PLB;
            const T* Pb = Tbuf + (slot * 3 + 0) * PLB;
            const T* Vb = Tbuf + (slot * 3 + 1) * PLB;
            const T* Xb = Tbuf + (slot * 3 + 2) * PLB;
            const i64 e0 = st_int + (i64)(K - 1) * nint2d;
            const int off = (int)(e0 & (i64)(PER16 - 1));
            // elements [0, head) and [tail0, nint2d) lie in 16-byte granules shared with a neighbouring plane
            int head = (PER16 - off) & (PER16 - 1);
            if (head > nint2d) head = nint2d;
            int tail0 = nint2d - (int)((e0 + nint2d) & (i64)(PER16 - 1));
            if (tail0 < head) tail0 = head;
            const T* dcls = dtab + (K % P) * P * P;
            T* rplane = ring + ((kb_base + K) % RB) * PLANE;
            // All four warps take part in every plane, so a warp revisits a transient slot only after its own
            // arrival on `tupd` for the slot's previous plane: it is never two phases ahead of the barrier (phase
            // parity only tells "this phase" from "the previous one"; with whole planes per warp this was a race,
            // profiles/r02_notes.md).
            mbar_wait(&H.tfull[slot], (q / NT) & 1);
            B2_TOC(tu, 1);
            // 16-byte granules of the staged plane (buffer index bi = off + e).  Granules [g_lo, g_hi) lie
            // fully inside the plane: 128-bit shared-memory loads, 128-bit global stores, no per-element
            // checks.  The (at most two) partial granules at the ends go element by element.
            const int g_lo = off ? 1 : 0, g_hi = (off + tail0) / PER16;
            const int lane = ut & 31;
            // all four warps work on every plane: a transient slot is held for a quarter of the time
            constexpr int GSTR = NUPD;
            const int gl0 = ut;
            auto update_plane = [&](auto xm_) {
              constexpr int XM = decltype(xm_)::value;
              struct alignas(16) Vec { T v[PER16]; };
              auto pre = [&](T& r, T& p, T& x, T v, T m) {  // solvers.py:660-690 on one entry
                if (XM == 2) x += xc1 * p + xc2 * (p - m * r);
                else if (XM == 1) x += xc1 * p;
                r -= am1 * v;
                p = m * r + bm1 * p;
                const double rd = (double)r, mr = (double)m * rd;
                ls0 += rd * rd;
                ls4 += rd * mr;
              };
              const Vec* Rv = reinterpret_cast<const Vec*>(Rb);
              const Vec* Vv = reinterpret_cast<const Vec*>(Vb);
              const Vec* Pq = reinterpret_cast<const Vec*>(Pb);
              const Vec* Xv = reinterpret_cast<const Vec*>(Xb);
              Vec* Rg = reinterpret_cast<Vec*>(R + (e0 - off));  // 16-byte aligned global granules
              Vec* Pg = reinterpret_cast<Vec*>(Pv + (e0 - off));
              Vec* Xg = reinterpret_cast<Vec*>(X + (e0 - off));
              const unsigned short* it0 = itab - off;
              constexpr int UNR = XM ? MFCG_B2_UNRX : MFCG_B2_UNR;
              constexpr int LOOPUNR = MFCG_B2_LOOPUNR;
              int round = 0;
#pragma unroll LOOPUNR
              for (int g0 = g_lo + gl0; g0 < g_hi; g0 += UNR * GSTR, round += UNR) {
                Vec rr[UNR], vv[UNR], pq[UNR], xx[UNR];
                unsigned tt[UNR][PER16];
                T mm[UNR][PER16];
                // warp-uniform: some lane of this warp has a granule in the next round
                const bool more = g0 - lane + GSTR < g_hi;
#pragma unroll
                for (int c = 0; c < UNR; ++c) {
                  if (c > 0 && !more) break;
                  const int gq = g0 + c * GSTR < g_hi ? g0 + c * GSTR : g0;  // the tail repeats granule g0 (discarded)
                  rr[c] = Rv[gq]; vv[c] = Vv[gq]; pq[c] = Pq[gq];
                  if (XM) xx[c] = Xv[gq];
                  if (CACHED) {
                    const int j = UNR == 2 ? c : round;  // planes have at most two rounds here
                    const unsigned pk = off ? (j ? tcache[1][1] : tcache[1][0]) : (j ? tcache[0][1] : tcache[0][0]);
                    tt[c][0] = pk & 0xffffu;
                    tt[c][PER16 - 1] = pk >> 16;
                  } else {
#pragma unroll
                    for (int w = 0; w < PER16; ++w) tt[c][w] = (MFCG_B2_SKIP & 64) ? 0u : it0[gq * PER16 + w];
                  }
#pragma unroll
                  for (int w = 0; w < PER16; ++w) mm[c][w] = (MFCG_B2_SKIP & 64) ? (T)1 : dcls[tt[c][w] >> 10];
                }
#pragma unroll
                for (int c = 0; c < UNR; ++c) {
                  const int gq = g0 + c * GSTR;
                  if (c > 0 && gq >= g_hi) break;
#pragma unroll
                  for (int w = 0; w < PER16; ++w) {
                    const T m = mm[c][w];
                    T xdummy = (T)0;
                    pre(rr[c].v[w], pq[c].v[w], XM ? xx[c].v[w] : xdummy, vv[c].v[w], m);
                    MFCG_CHECK((int)(tt[c][w] & 1023u) < PLANE);
                    if (!(MFCG_B2_SKIP & 2)) rplane[tt[c][w] & 1023u] = pq[c].v[w];
                  }
                  *reinterpret_cast<Vec*>(Rb + gq * PER16) = rr[c];  // r' stays staged for the gather's sums
                  if (MFCG_B2_SKIP & 1) continue;
                  MFCG_CHECK(e0 - off + (i64)gq * PER16 >= 0 && e0 - off + (i64)(gq + 1) * PER16 <= n_int);
                  Rg[gq] = rr[c];
                  Pg[gq] = pq[c];
                  if (XM) Xg[gq] = xx[c];
                }
              }
              // partial granules: element e of the head [0, head) or the tail [tail0, nint2d)
              const int npart = head + (nint2d - tail0);
              if (lane < npart && uw == NUPD / 32 - 1) {
                const int e = lane < head ? lane : tail0 + (lane - head);
                const unsigned t = itab[e];
                const T m = dcls[t >> 10];
                T r = Rb[off + e], p = Pb[off + e], x = XM ? Xb[off + e] : (T)0;
                pre(r, p, x, Vb[off + e], m);
                rplane[t & 1023u] = p;
                Rb[off + e] = r;
                MFCG_CHECK(e0 + e >= 0 && e0 + e < n_int);
                R[e0 + e] = r;
                Pv[e0 + e] = p;
                if (XM) X[e0 + e] = x;
              }
            };
            if (MFCG_B2_SKIP & 4) {}
            else if (xmode == 0) update_plane(std::integral_constant<int, 0>());
            else if (xmode == 1) update_plane(std::integral_constant<int, 1>());
            else update_plane(std::integral_constant<int, 2>());
            mbar_arrive(&H.tupd[slot]);  // the transient slot (p, v, x) has been read
            B2_TOC(tu, 2);
          }
        B2_TOC(tu, 4);
        if (L == bcz - 1) {  // handed over with the brick's last layer
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            ls0 += __shfl_xor_sync(0xffffffffu, ls0, o);
            ls4 += __shfl_xor_sync(0xffffffffu, ls4, o);
          }
          if ((ut & 31) == 0) { H.lsum[gl & 3][uw][0] = ls0; H.lsum[gl & 3][uw][1] = ls4; }
        }
        mbar_arrive(&H.lfull[gl & 3]);
        B2_TOC(tu, 5);
      }
    } else if constexpr (ROLE == 0) {
      // ================================ plane sweeps (warpgroup 0) ================================
      // Brick-boundary values of p' (pre-updated by k_pre, unchanged during this launch) go straight into the
      // ring with 8-byte cp.async, one layer ahead of the sweeps: these warps idle while the update warps work.
      i64* s27 = H.st27[1];
      named_barrier<6, NS1>();
      if (tid < 27) s27[tid] = entity(tid);
      named_barrier<6, NS1>();
      const int nperim = fp - nint2d;
      const int n_in_c = bcx * (P - 1) * bcy * (P - 1);
      // this thread's brick-boundary position of a lattice plane (the same for every plane of the brick)
      int pe2 = 0, pcw = 0, po2 = 0, ppstride = 0;
      if (tid < nperim) {
        const uint2 d = gtab[n_in_c + tid];
        pe2 = (int)((d.x >> 19) & 15u); pcw = (int)(d.y & 1023u); po2 = (int)((d.y >> 10) & 4095u);
        const unsigned sel = d.y >> 22;
        ppstride = ((sel & 1u) ? Lx - 1 : 1) * ((sel & 2u) ? Ly - 1 : 1);
      }
      const T* src1 = Pv + (s27[pe2 + 9] + po2 - ppstride);  // planes 0 < K < Lz: src1[ppstride * K]
      const unsigned ring_pos = smem_u32(ring + pcw);
      const bool bnd_xy = mx == 0 || mx == g.mb[0] - 1 || my == 0 || my == g.mb[1] - 1;
      // ZERO = false: issue the copies of layer L, return the Dirichlet bits of this thread's values
      // (bits 0..P: planes, 8.., 16..: bottom / top face); ZERO = true: zero the flagged values (operator.py:341-342)
      auto boundary = [&](int L, auto zero_c, unsigned bits, unsigned (&pm)[P + 1]) -> unsigned {
        constexpr bool ZERO = decltype(zero_c)::value;
        const int k0 = L == 0 ? 0 : 1;
        // Dirichlet DoFs lie on the domain boundary (enforced at operator creation): only bricks that touch it
        // need the mask bytes
        const bool need_mask = bnd_xy || (mz == 0 && L == 0) || (mz == g.mb[2] - 1 && L == bcz - 1);
        unsigned out = 0;
        if (tid < nperim) {
          const int nk = P + 1 - k0;
          int K = L * P + k0;
          int slot = (kb_base + K) % RB;
          const T* src = src1 + (i64)ppstride * K;  // planes strictly inside the brick: one stride apart
#pragma unroll
          for (int kk = 0; kk < P + 1; ++kk, ++K, src += ppstride, slot = slot + 1 == RB ? 0 : slot + 1) {
            if (kk >= nk) break;
            if (ZERO) {
              if (bits & (1u << kk)) ring[slot * PLANE + pcw] = (T)0;
              continue;
            }
            const T* sp = src;
            if (K == 0 || K == Lz) sp = Pv + s27[pe2 + (K == 0 ? 0 : 18)] + po2;  // the brick's bottom / top plane
            MFCG_CHECK(sp - Pv >= n_int && sp - Pv < g.n_dofs && pcw < PLANE && K <= Lz);
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(ring_pos + (unsigned)(slot * PLANE * (int)sizeof(T))),
                         "l"(sp), "n"((int)sizeof(T)) : "memory");
            // the mask byte stays an outstanding load: it is folded into the flag bits after this layer's sweeps
            if (need_mask) pm[kk] = g.mask[(sp - Pv) - n_int];
          }
        }
        // the brick's bottom / top face interiors (first / last layer only): contiguous in memory
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (side == 0 ? (L != 0) : (L != bcz - 1)) continue;
          const i64 fb = s27[side == 0 ? 4 : 22];
          T* pl = ring + ((kb_base + (side == 0 ? 0 : Lz)) % RB) * PLANE;
          const bool face_mask = side == 0 ? mz == 0 : mz == g.mb[2] - 1;  // the face lies on the domain boundary
          int cnt = 8 + 8 * side;
          for (int it = tid; it < nint2d; it += NS1, ++cnt) {
            T* dstp = pl + (itab[it] & 1023u);
            if (ZERO) {
              if (bits & (1u << cnt)) *dstp = (T)0;
              continue;
            }
            MFCG_CHECK(fb + it >= n_int && fb + it < g.n_dofs);
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dstp)), "l"(Pv + fb + it),
                         "n"((int)sizeof(T)) : "memory");
            if (face_mask) out |= (unsigned)(g.mask[fb + it - n_int] & 1) << cnt;
          }
        }
        if (!ZERO) asm volatile("cp.async.commit_group;" ::: "memory");
        return out;
      };
      static_assert((P * G2::BX + 1) * 2 + (P * G2::BY - 1) * 2 <= NS1, "one brick-boundary position per thread");
      static_assert(((P * G2::BX - 1) * (P * G2::BY - 1) + NS1 - 1) / NS1 <= 8, "face bits");
      // the ring planes a layer overwrites were last read by the gather RLAYERS layers back; that gather had
      // finished before these warps were let into the layer before this one (tile barrier), so no wait is needed
      // beyond the check below (immediate)
      auto ring_free = [&](int gq) {
        if (gq >= G2::RLAYERS) mbar_wait(&H.ldone[(gq - G2::RLAYERS) & 3], ((gq - G2::RLAYERS) >> 2) & 1);
      };
      unsigned pm[P + 1];
      auto fold = [&](unsigned b) {  // Dirichlet flags of the values issued last
#pragma unroll
        for (int kk = 0; kk < P + 1; ++kk) {
          pin_value(pm[kk]);
          b |= (pm[kk] & 1u) << kk;
          pm[kk] = 0u;
        }
        return b;
      };
#pragma unroll
      for (int kk = 0; kk < P + 1; ++kk) pm[kk] = 0u;
      ring_free(g_base);
      unsigned bits_cur = fold(boundary(0, std::false_type(), 0u, pm)), bits_next = 0;
      for (int L = 0; L < bcz; ++L) {
        const int gl = g_base + L;
        const int sl0 = (kb_base + L * P) % RB;
        B2_TIC(tm);
        if (L + 1 < bcz) {
          ring_free(gl + 1);
          B2_TOC(tm, 5);
          bits_next = boundary(L + 1, std::false_type(), 0u, pm);
          B2_TOC(tm, 4);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        if (bits_cur) boundary(L, std::true_type(), bits_cur, pm);
        B2_TOC(tm, 5);
        named_barrier<6, NS1>();  // every thread's values of layer L have landed
#ifdef MFCG_TIMING
        { volatile double* vv_ = &H.bsum[0]; (void)*vv_; }  // the barrier blocks at the first dependent access
        { long long n__ = clock64(); tacc6 += (unsigned long long)(n__ - tm); tm = n__; }
#endif
        mbar_wait(&H.lfull[gl & 3], (gl >> 2) & 1);
        B2_TOC(tm, 0);
        // ---- stage 1: thread = (cell, z plane k); the plane goes to registers, x and y sweeps there:
        //      c = My Mx u -> A tile,  d = (gy Ky Mx + My gx Kx) u -> B tile
        bool tiles_free = false;
#pragma unroll 1
        for (int t = tid; t < NCELL * N; t += NS1) {
          const int cell = t % NCELL, k = t / NCELL;
          T a[N][N], bq[N][N];
          const bool has_cell = cell < bcx * bcy && !(MFCG_B2_SKIP & 32);
          if (has_cell) {
            const int ccy = cell / bcx, ccx = cell - ccy * bcx;
            int slot = sl0 + k;
            if (slot >= RB) slot -= RB;
            const T* rp = ring + slot * PLANE + ccy * (P * WX + SK) + ccx * P;
#pragma unroll
            for (int j = 0; j < N; ++j) {
              T u[N], e[HE], o[HE], se[HE], so[HE];
#pragma unroll
              for (int i = 0; i < N; ++i) u[i] = rp[j * WX + (j == P ? SK : 0) + i];
              eo_split<N>(u, e, o);
#pragma unroll
              for (int i = 0; i < HE; ++i) { se[i] = 0; so[i] = 0; }
              eo_mul<N>(tab.Me, tab.Mo, e, o, se, so);
              eo_join<N>(se, so, a[j]);
#pragma unroll
              for (int i = 0; i < HE; ++i) { se[i] = 0; so[i] = 0; }
              eo_mul<N>(tab.Ke[0], tab.Ko[0], e, o, se, so);
              eo_join<N>(se, so, bq[j]);
            }
#pragma unroll
            for (int i = 0; i < N; ++i) {
              T col[N], ea[HE], oa[HE], eb[HE], ob[HE], se[HE], so[HE], out[N];
#pragma unroll
              for (int j = 0; j < N; ++j) col[j] = a[j][i];
              eo_split<N>(col, ea, oa);
#pragma unroll
              for (int j = 0; j < N; ++j) col[j] = bq[j][i];
              eo_split<N>(col, eb, ob);
#pragma unroll
              for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
              eo_mul<N>(tab.Ke[1], tab.Ko[1], ea, oa, se, so);  // gy K a
              eo_mul<N>(tab.Me, tab.Mo, eb, ob, se, so);        // + M b
              eo_join<N>(se, so, out);
#pragma unroll
              for (int j = 0; j < N; ++j) bq[j][i] = out[j];
#pragma unroll
              for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
              eo_mul<N>(tab.Me, tab.Mo, ea, oa, se, so);        // c = M a
              eo_join<N>(se, so, out);
#pragma unroll
              for (int j = 0; j < N; ++j) a[j][i] = out[j];
            }
          }
          B2_TOC(tm, 1);
          if (!tiles_free) {  // the gather of the previous layer has read the tiles
            if (gl > 0) named_barrier<4, NS1 + NLM>();
            tiles_free = true;
          }
          B2_TOC(tm, 2);
          if (has_cell) {
            T* At = A + cell * TILE + k * PSTR;
            T* Bt = Bs + cell * TILE + k * PSTR;
#pragma unroll
            for (int j = 0; j < N; ++j)
#pragma unroll
              for (int i = 0; i < N; ++i) {
                At[j * RS + i] = a[j][i];
                Bt[j * RS + i] = bq[j][i];
              }
          }
        }
        if (!tiles_free && gl > 0) named_barrier<4, NS1 + NLM>();
        named_arrive<3, NS1 + NLM>();  // tiles of layer gl written
        bits_cur = fold(bits_next);
        bits_next = 0u;
        B2_TOC(tm, 3);

      }
    } else {
      // ================================ z sweep + gather (warpgroups 1-2) ================================
      const int lt = tid - T_LM;
      i64* s27 = H.st27[0];
      if (lt < 27) s27[lt] = entity(lt);
      for (int i = lt; i < PLANE; i += NLM) carry[i] = (T)0;
      named_barrier<1, NLM>();
      const i64 st_int = s27[13];
      double s1 = 0, s2 = 0, s3 = 0, s5 = 0, s6 = 0;
      for (int L = 0; L < bcz; ++L) {
        const int gl = g_base + L;
        const int sl0 = (kb_base + L * P) % RB;
        B2_TIC(tm);
        named_barrier<3, NS1 + NLM>();  // tiles of layer gl written (the plane-sweep group waited for lfull)
#ifdef MFCG_TIMING
        { volatile double* vv_ = &H.bsum[0]; (void)*vv_; }  // the barrier blocks at the first dependent access
#endif
        B2_TOC(tm, 0);
        if (lt == 0 && L == bcz - 1) {  // r.r and r.Mr of the brick from the update warps
          double a0_ = 0.0, a4_ = 0.0;
          for (int w = 0; w < NUPD / 32; ++w) { a0_ += H.lsum[gl & 3][w][0]; a4_ += H.lsum[gl & 3][w][1]; }
          H.bsum[0] = a0_; H.bsum[1] = a4_;
        }

        // ---- stage 2: z sweep per (cell, column): out = M d + gz K c, written over c
#pragma unroll 1
        for (int t = lt; t < ((MFCG_B2_SKIP & 16) ? 0 : NCELL * N * N); t += NLM) {
          const int cell = t % NCELL, l = t / NCELL;
          if (cell >= bcx * bcy) continue;
          T* ac = A + cell * TILE + l;
          const T* bc = Bs + cell * TILE + l;
          T ca[N], cb[N], ec[HE], oc[HE], ed[HE], od[HE], se[HE], so[HE], out[N];
#pragma unroll
          for (int k = 0; k < N; ++k) { ca[k] = ac[k * PSTR]; cb[k] = bc[k * PSTR]; }
          eo_split<N>(ca, ec, oc);
          eo_split<N>(cb, ed, od);
#pragma unroll
          for (int i2 = 0; i2 < HE; ++i2) { se[i2] = 0; so[i2] = 0; }
          eo_mul<N>(tab.Ke[2], tab.Ko[2], ec, oc, se, so);  // gz K c
          eo_mul<N>(tab.Me, tab.Mo, ed, od, se, so);        // + M de
          eo_join<N>(se, so, out);
#pragma unroll
          for (int k = 0; k < N; ++k) ac[k * PSTR] = out[k];
        }
        B2_TOC(tm, 1);
        named_barrier<1, NLM>();
        B2_TOC(tm, 3);

        // ---- gather per lattice point (fixed order, no shared-memory atomics), v out, post sums
        const T* Rl = Rbuf + (gl % NRL) * P * PLB;  // r' of the planes this layer finishes: K = L*P + k, k < P
        int offk[P];
#pragma unroll
        for (int k = 0; k < P; ++k) offk[k] = (int)((st_int + (i64)(L * P + k - 1) * nint2d) & (i64)(PER16 - 1));
        int rso[P];  // ring plane of k
#pragma unroll
        for (int k = 0; k < P; ++k) rso[k] = ((sl0 + k) % RB) * PLANE;
        // the five sums of a finished DoF, on r', p' and 1/diag that stayed on chip (solvers.py:692-698)
        auto post = [&](T r_, T p_, T m_, T v_) {
          const double r = (double)r_, p = (double)p_, m = (double)m_, v = (double)v_;
          const double mv = m * v;
          s1 += p * v; s2 += r * v; s3 += v * v; s5 += r * mv; s6 += v * mv;
        };
        for (int rem = lt; rem < ((MFCG_B2_SKIP & 8) ? 0 : fp); rem += NLM) {
          const uint2 d = gtab[rem];
          const int base = (int)(d.x & 16383u), cw = (int)(d.y & 1023u), o2 = (int)((d.y >> 10) & 4095u);
          const int cls = (int)((d.x >> 23) & 127u);
          const bool edge = (d.x >> 18) & 1u;
          // all shared-memory loads of the point first (independent, in flight together), then the stores
          T sum[P + 1];
          if (((d.x >> 14) & 31u) == 1u) {
            // strictly inside one cell in x and y: one contribution per plane
            MFCG_CHECK(base + P * PSTR < NCELL * TILE && cw < PLANE);
#pragma unroll
            for (int k = 0; k <= P; ++k) sum[k] = A[base + k * PSTR];
          } else {
            const int o11 = (d.x & (1u << 14)) ? base : -1;
            const int o10 = (d.x & (1u << 15)) ? base - TILE + P : -1;
            const int o01 = (d.x & (1u << 16)) ? base - bcx * TILE + P * RS : -1;
            const int o00 = (d.x & (1u << 17)) ? base - (bcx + 1) * TILE + P * RS + P : -1;
#pragma unroll
            for (int k = 0; k <= P; ++k) {
              T acc = 0;
              if (o00 >= 0) acc += A[o00 + k * PSTR];
              if (o01 >= 0) acc += A[o01 + k * PSTR];
              if (o10 >= 0) acc += A[o10 + k * PSTR];
              if (o11 >= 0) acc += A[o11 + k * PSTR];
              sum[k] = acc;
            }
          }
          sum[0] += carry[cw];
          if (!edge) {
            MFCG_CHECK(offk[P - 1] + o2 < PLB);
            // brick-interior DoFs of the column: planes K = L*P + k
            const i64 gi0 = st_int + o2 + (i64)nint2d * (L * P - 1);
            if (L == 0) atomicAdd(&V[s27[4] + o2], sum[0]);  // the brick's bottom face is shared
            else {
              MFCG_CHECK(gi0 >= 0 && gi0 < n_int);
              V[gi0] = sum[0];
              post(Rl[offk[0] + o2], ring[rso[0] + cw], dtab[cls], sum[0]);
            }
#pragma unroll
            for (int k = 1; k < P; ++k) {
              MFCG_CHECK(gi0 + (i64)k * nint2d >= 0 && gi0 + (i64)k * nint2d < n_int);
              V[gi0 + (i64)k * nint2d] = sum[k];
              post(Rl[k * PLB + offk[k] + o2], ring[rso[k] + cw], dtab[k * P * P + cls], sum[k]);
            }
            if (L < bcz - 1) carry[cw] = sum[P];
            else atomicAdd(&V[s27[22] + o2], sum[P]);  // top face
          } else {
            // brick-boundary point: shared DoFs on every plane (k_pre / k_post own their vector updates);
            // constrained rows receive garbage here, k_post restores v_c = p_c
            const int e2 = (int)((d.x >> 19) & 15u);
            const unsigned sel = d.y >> 22;
            const int pstride = ((sel & 1u) ? Lx - 1 : 1) * ((sel & 2u) ? Ly - 1 : 1);
#pragma unroll
            for (int k = 0; k <= P; ++k) {
              if (k == P && L < bcz - 1) {
                carry[cw] = sum[k];
                continue;
              }
              const int K = L * P + k;
              const int ez = K == 0 ? 0 : (K == Lz ? 2 : 1);
              const i64 gi = s27[e2 + 9 * ez] + o2 + (ez == 1 ? (i64)pstride * (K - 1) : 0);
              MFCG_CHECK(gi >= n_int && gi < g.n_dofs);
              atomicAdd(&V[gi], sum[k]);
            }
          }
        }
        mbar_arrive(&H.ldone[gl & 3]);
        named_arrive<4, NS1 + NLM>();  // tiles free for the next layer
        B2_TOC(tm, 2);
      }
      // brick sums, fixed order (deterministic)
      {
        double sm[7] = {0.0, s1, s2, s3, 0.0, s5, s6};
        if (lt == 0) { sm[0] = H.bsum[0]; sm[4] = H.bsum[1]; H.bsum[0] = 0.0; H.bsum[1] = 0.0; }
        warp_reduce7(sm);
        named_barrier<1, NLM>();  // the previous brick's row has been written
        if ((lt & 31) == 0)
#pragma unroll
          for (int qq = 0; qq < 7; ++qq) H.red[lt >> 5][qq] = sm[qq];
        named_barrier<1, NLM>();
        if (lt < 7) {
          double acc = 0.0;
          for (int w = 0; w < NLM / 32; ++w) acc += H.red[w][lt];
          partials[(i64)b * 8 + lt] = acc;
        }
      }
    }
    g_base += bcz;
    q_base += nplanes;
    kb_base = (kb_base + Lz + 1) % RB;
  }
#ifdef MFCG_TIMING
  if (tid == 0 || tid == T_LM || tid == T_PROD || tid == T_UPD)
    for (int i = 0; i < (tid == T_UPD ? 6 : 4); ++i)
      atomicAdd(&g_phase_cycles[(tid == 0 ? 0 : (tid == T_LM ? 4 : (tid == T_PROD ? 8 : 12))) + i], tacc[i]);
  if (tid == 0) {  // plane-sweep warps, brick-boundary fetch: issue, ring check + landing + zeroing, barrier
    atomicAdd(&g_phase_cycles[18], tacc[4]);
    atomicAdd(&g_phase_cycles[19], tacc[5]);
    atomicAdd(&g_phase_cycles[20], tacc6);
  }
#endif
  };
  // register re-allocation between the warpgroups: the plane sweeps hold 2 (p+1)^2 values per thread
  if (tid < T_LM) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(G2::REG_S1));
    if (tid < T_PROD) run_role(std::integral_constant<int, 0>());
    else run_role(std::integral_constant<int, 1>());  // the warpgroup's fourth warp has no planes: producer
  } else if (tid < T_UPD) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(G2::REG_LIGHT));
    run_role(std::integral_constant<int, 3>());
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(G2::REG_UPD));
    run_role(std::integral_constant<int, 2>());
  }
}

}  // namespace mfcg
