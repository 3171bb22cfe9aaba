// tl_kernels.cuh — device kernels of the two-level heat solve (sm_100a, fp64).
//
//   k_pcg        persistent cooperative kernel: RHS build (mass, Gaussian load,
//                dense extra load, Dirichlet lift) + Jacobi-PCG mirroring scipy's
//                cg + true-residual check + Dirichlet re-imposition.
//                Replaces fem.assemble_system + constrained + solve_linear
//                (lpbfsim/fem.py:129-194, 89-105, 271-298) for one solve.
//   k_interp     Kuhn-P1 interpolation of the global field at local nodes
//                (Mesh.interpolate / InterfaceGamma.trace_of, mesh.py:358-361,471-474;
//                relocate_local re-interpolation, scanpath.py:243-248).
//   k_interp_pts same at arbitrary points.
//   k_deposit    SweptTrackDeposit.load scatter (sources.py:164-172), deterministic.
//   k_melt       max T and melt-node count (T > T_liquidus) of one field.
//   k_flush      writes a buffer larger than L2 (benchmark hygiene).
//   k_trans_entries / k_trans_segsum  transmission_load (twolevel.py:159-183): the
//                interface facets' flux-jump functional on global test functions,
//                scattered deterministically (stable key sort + ordered segment sums).
//   k_mass_norms discrete L2 norms v^T M v with the P1 mass matrix (fem.mass_matrix,
//                fem.py:434-446) of a field difference and of the reference field:
//                the metrics of metrics.error_metrics (metrics.py:123-165).
#pragma once

#include <cooperative_groups.h>

#include "tl_grid.cuh"

namespace cg = cooperative_groups;

namespace tl {

constexpr int kTPB = 512;                  // threads per block of k_pcg
constexpr int kMaxTab = 4096;              // Gaussian table entries per axis (cells)
// length (doubles) of PcgParams::part: resident slots (< 4096), k_s_cg partials at 4096,
// k_t_cg counters at 2048 and item partials at 4096 + 3 * kTMaxItems
constexpr int kPartLen = 4096 + 3 * 16384 + 1024;

// 4-point tet rule (mesh.py:116-128) and the six per-axis fractional offsets a
// Kuhn-tet quadrature point can take inside its cell: {b, 2b, 3b, a, a+b, a+2b}.
#define TL_QA ((5.0 + 3.0 * 2.23606797749978969640917366873127623544) / 20.0)
#define TL_QB ((5.0 - 2.23606797749978969640917366873127623544) / 20.0)

// For permutation index pi (itertools.permutations order) and quadrature point q,
// the offset index (into the six values) along x, y, z.
__constant__ int8_t c_qoff[6][4][3] = {
    {{2, 1, 0}, {5, 1, 0}, {5, 4, 0}, {5, 4, 3}}, {{2, 0, 1}, {5, 0, 1}, {5, 0, 4}, {5, 3, 4}},
    {{1, 2, 0}, {1, 5, 0}, {4, 5, 0}, {4, 5, 3}}, {{0, 2, 1}, {0, 5, 1}, {0, 5, 4}, {3, 5, 4}},
    {{1, 0, 2}, {1, 0, 5}, {4, 0, 5}, {4, 3, 5}}, {{0, 1, 2}, {0, 1, 5}, {0, 4, 5}, {3, 4, 5}}};
// Tets of a cell containing its corner with offset bits (bx | by<<1 | bz<<2): list of
// (perm index, local vertex index j).  Offsets 0 and 7 lie on all six tets.
__constant__ int8_t c_inc_n[8] = {6, 2, 2, 2, 2, 2, 2, 6};
__constant__ int8_t c_inc[8][6][2] = {
    {{0, 0}, {1, 0}, {2, 0}, {3, 0}, {4, 0}, {5, 0}}, {{0, 1}, {1, 1}},
    {{2, 1}, {3, 1}}, {{0, 2}, {2, 2}}, {{4, 1}, {5, 1}}, {{1, 2}, {4, 2}},
    {{3, 2}, {5, 2}}, {{0, 3}, {1, 3}, {2, 3}, {3, 3}, {4, 3}, {5, 3}}};

struct Gauss {
    double peak, radius, depth, center[3];
    int on;
};

struct SolveInfoDev {
    int iterations, status;
    double bnorm, rnorm, true_resid;
};

struct PcgParams {
    Grid g;
    double cbase[3];     // kappa V / (6 h_a^2)
    double mbase;        // (rho c / dt) V / 24
    // inputs
    double* T;           // T_old in, solution out (in place)
    const double* gA;    // Dirichlet values (1-w) gA + w gB, or g_const if gA == nullptr
    const double* gB;
    double w, g_const;
    const double* load;  // dense extra load or nullptr
    // streaming solves of a run: Gaussian load precomputed by k_gauss_loads, dense over the
    // box bbox = [i0, i1) x [j0, j1) x [k0, k1) (device memory; x fastest), or nullptr
    const double* bload;
    const int* bbox;
    Gauss src;
    // workspace
    double *b, *r, *p0, *p1, *q;
    double* part;        // [4][gridDim]
    double rtol;
    int maxiter;
    SolveInfoDev* info;
    int light_rhs;       // k_t_cg path: k_s_rhs writes b only (r0 = b and x0 = 0 are implied)
    int snake;           // k_s_cg: sweep B walks the grid top-down (TLGPU_SNAKE, tl_stream.cuh)
    unsigned long long* prof;   // TLGPU_PROF=1: k_s_cg %globaltimer stamps of iteration 3 (slot 1024 + 16 CTA + e)
};

__device__ __forceinline__ unsigned long long timer_ns() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum of NV values; result valid in thread 0 (the trailing barrier
// measured faster than leaving the other warps to wait inside grid.sync).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) smem[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = lane < nw ? smem[k * 32 + lane] : 0.0;
            v[k] = warp_sum(s);
        }
    }
    __syncthreads();
}

// Fixed-order sum of the per-block partials written before the last grid.sync.
// Every block computes bitwise the same totals (commutative butterfly).
template <int NV>
__device__ __forceinline__ void grid_sum(const double* part, const int (&slot)[NV], int G,
                                         double* smem_out) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const double* p = part + slot[k] * G;
            double s = 0.0;
            for (int b = lane; b < G; b += 32) s += __ldcg(p + b);
            s = warp_sum(s);
            if (lane == 0) smem_out[k] = s;
        }
    }
    __syncthreads();
}

constexpr int kResMaxBlocks = 320;       // grid-reduction capacity (CTAs)

// Fixed-order, load-parallel sum of G <= MAXG partials (all blocks agree bitwise).
// All NV x ceil(G/32) loads of a lane are issued before any add: one L2 round trip.
template <int NV, int MAXG = 160>
__device__ __forceinline__ void grid_sum_fast(const double* part, const int (&slot)[NV], int G,
                                              double* smem_out) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        constexpr int PL = MAXG / 32;
        double v[NV][PL];
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int t = 0; t < PL; ++t) {
                const int b = lane + 32 * t;
                v[k][t] = b < G ? __ldcg(part + slot[k] * G + b) : 0.0;
            }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
#pragma unroll
            for (int t = 0; t < PL; ++t) s += v[k][t];
            s = warp_sum(s);
            if (lane == 0) smem_out[k] = s;
        }
    }
    __syncthreads();
}

// Dirichlet value at node p.
__device__ __forceinline__ double dirichlet_value(const PcgParams& P, int p) {
    if (P.gA == nullptr) return P.g_const;
    return __dadd_rn(__dmul_rn(1.0 - P.w, P.gA[p]), __dmul_rn(P.w, P.gB[p]));
}

// Dirichlet lift of a free row (SparseSystem.constrained, fem.py:96-101):
// -sum_{q in D} A_pq g_q with A_pq = -c_pq.
__device__ __forceinline__ double dirichlet_lift(const PcgParams& P, const ClassTable& T, int p, int i, int j,
                                                 int k, int cls) {
    const Grid& g = P.g;
    const int sy = g.NX, sz = g.NX * g.NY;
    double lift = 0.0;
    if (i > 0 && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i - 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dirichlet_value(P, p - 1);
    if (i < g.nc[0] && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dirichlet_value(P, p + 1);
    if (j > 0 && T.nd[cls + 3 * (axis_class(j - 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dirichlet_value(P, p - sy);
    if (j < g.nc[1] && T.nd[cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dirichlet_value(P, p + sy);
    if (k > 0 && T.nd[cls + 9 * (axis_class(k - 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dirichlet_value(P, p - sz);
    if (k < g.nc[2] && T.nd[cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dirichlet_value(P, p + sz);
    return lift;
}

// Gaussian nodal load: sum over incident Kuhn tets of
// (V/24) * (b * S_tet + (a - b) * Q_own), Q = peak * Ex * Ey * Ez from per-axis tables
// tab[axis][cell * 6 + offset] (peak and V/24 folded into the z table).
__device__ double gaussian_node(const Grid& g, const double* tx, const double* ty,
                                const double* tz, int i, int j, int k) {
    double F = 0.0;
#pragma unroll
    for (int bz = 0; bz < 2; ++bz) {
        const int cz = k - bz;
        if (cz < 0 || cz >= g.nc[2]) continue;
#pragma unroll
        for (int by = 0; by < 2; ++by) {
            const int cy = j - by;
            if (cy < 0 || cy >= g.nc[1]) continue;
#pragma unroll
            for (int bx = 0; bx < 2; ++bx) {
                const int cx = i - bx;
                if (cx < 0 || cx >= g.nc[0]) continue;
                const double* ex = tx + cx * 6;
                const double* ey = ty + cy * 6;
                const double* ez = tz + cz * 6;
                const int off = bx | (by << 1) | (bz << 2);
                const int ninc = c_inc_n[off];
                for (int t = 0; t < ninc; ++t) {
                    const int pi = c_inc[off][t][0], jv = c_inc[off][t][1];
                    double S = 0.0, Qj = 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double Q = ex[c_qoff[pi][q][0]] * ey[c_qoff[pi][q][1]] * ez[c_qoff[pi][q][2]];
                        S += Q;
                        Qj = (q == jv) ? Q : Qj;
                    }
                    F += TL_QB * S + (TL_QA - TL_QB) * Qj;
                }
            }
        }
    }
    return F;
}

}  // namespace tl
#include "tl_gauss_gen.cuh"
namespace tl {

// Same load, branch-free: the 2 x 6 table values per axis in registers (zero for
// cells outside the grid) and the 96 terms of tl_gauss_gen.cuh.
__device__ __forceinline__ double gaussian_node_fast(const Grid& g, const double* tx, const double* ty,
                                                     const double* tz, int i, int j, int k) {
    double X[2][6], Y[2][6], Z[2][6];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const bool vx = (i - b) >= 0 && (i - b) < g.nc[0];
        const bool vy = (j - b) >= 0 && (j - b) < g.nc[1];
        const bool vz = (k - b) >= 0 && (k - b) < g.nc[2];
#pragma unroll
        for (int o = 0; o < 6; ++o) {
            X[b][o] = vx ? tx[(i - b) * 6 + o] : 0.0;
            Y[b][o] = vy ? ty[(j - b) * 6 + o] : 0.0;
            Z[b][o] = vz ? tz[(k - b) * 6 + o] : 0.0;
        }
    }
    return gauss_terms(X, Y, Z);
}

// Per-node-index upper bound of the Gaussian table factors: m[idx] = max over the
// (up to) two cells idx-1, idx and the six offsets.  F_p <= 24 mx[i] my[j] mz[k]
// (the 24 incident tets each weigh their four points by a + 3b = 1).
__host__ __device__ inline int gauss_smem_len(const Grid& g) {
    return 6 * (g.nc[0] + g.nc[1] + g.nc[2]) + (g.nc[0] + 1) + (g.nc[1] + 1) + (g.nc[2] + 1);
}

__device__ inline void build_gauss_bounds(const Grid& g, const double* tx, const double* ty,
                                          const double* tz, double* mx, double* my, double* mz) {
    const int tot = g.NX + g.NY + g.NZ;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int a = 0, idx = e;
        if (idx >= g.NX) { idx -= g.NX; a = 1; if (idx >= g.NY) { idx -= g.NY; a = 2; } }
        const double* t = a == 0 ? tx : (a == 1 ? ty : tz);
        double m = 0.0;
        for (int c = idx - 1; c <= idx; ++c)
            if (c >= 0 && c < g.nc[a])
                for (int o = 0; o < 6; ++o) m = fmax(m, t[c * 6 + o]);
        (a == 0 ? mx : (a == 1 ? my : mz))[idx] = m;
    }
}

// b0 + F_p, skipping the 96-term evaluation when F_p cannot change b0: for
// 0 <= F < 2^-55 b0 the rounded sum is b0 exactly, so the result is bitwise the
// same as adding the evaluated load (the Gaussian is negligible far from the beam).
__device__ __forceinline__ double add_gaussian(double b0, const Grid& g, const double* tx,
                                               const double* ty, const double* tz, const double* mx,
                                               const double* my, const double* mz, int i, int j, int k) {
    const double bound = 24.0 * mx[i] * my[j] * mz[k];
    if (b0 > 0.0 && bound < b0 * 0x1p-55) return b0;
    return b0 + gaussian_node_fast(g, tx, ty, tz, i, j, k);
}

__device__ inline void build_gauss_tables(const Grid& g, const Gauss& s, double* tx, double* ty,
                                          double* tz) {
    const double fr[6] = {TL_QB, 2.0 * TL_QB, 3.0 * TL_QB, TL_QA, TL_QA + TL_QB, TL_QA + 2.0 * TL_QB};
    const double V24 = g.h[0] * g.h[1] * g.h[2] / 24.0;
    const int tot = 6 * (g.nc[0] + g.nc[1] + g.nc[2]);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int a, rem = e;
        if (rem < 6 * g.nc[0]) a = 0;
        else if ((rem -= 6 * g.nc[0]) < 6 * g.nc[1]) a = 1;
        else { rem -= 6 * g.nc[1]; a = 2; }
        const int c = rem / 6, o = rem % 6;
        const double x = node_coord(g, a, c) + fr[o] * g.h[a];
        const double sc = (a == 2) ? s.depth : s.radius;
        const double t = (x - s.center[a]) / sc;
        double v = exp(-3.0 * (t * t));
        double* dst = a == 0 ? tx : (a == 1 ? ty : tz);
        if (a == 2) v *= s.peak * V24;
        dst[rem] = v;
    }
}

// Value of z = M r at node q (Jacobi), from its axis indices.
__device__ __forceinline__ int class_of(const Grid& g, int i, int j, int k) {
    return axis_class(i, g.nc[0]) + 3 * axis_class(j, g.nc[1]) + 9 * axis_class(k, g.nc[2]);
}

// y = (A_c v)_p for a free node p, v given by functor V(q, cls_q).
template <class F>
__device__ __forceinline__ double apply_free(const Grid& g, const ClassTable& T, int p, int i, int j,
                                             int k, int cls, double vp, F V) {
    double y = T.diag[cls] * vp;
    double s = 0.0;
    const int sy = g.NX, sz = g.NX * g.NY;
    // x neighbours
    {
        const double c = T.c[0][cls];
        double t = 0.0;
        if (i > 0) { int qc = cls - axis_class(i, g.nc[0]) + axis_class(i - 1, g.nc[0]); t += T.nd[qc] * V(p - 1, qc); }
        if (i < g.nc[0]) { int qc = cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0]); t += T.nd[qc] * V(p + 1, qc); }
        s += c * t;
    }
    {
        const double c = T.c[1][cls];
        double t = 0.0;
        if (j > 0) { int qc = cls + 3 * (axis_class(j - 1, g.nc[1]) - axis_class(j, g.nc[1])); t += T.nd[qc] * V(p - sy, qc); }
        if (j < g.nc[1]) { int qc = cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1])); t += T.nd[qc] * V(p + sy, qc); }
        s += c * t;
    }
    {
        const double c = T.c[2][cls];
        double t = 0.0;
        if (k > 0) { int qc = cls + 9 * (axis_class(k - 1, g.nc[2]) - axis_class(k, g.nc[2])); t += T.nd[qc] * V(p - sz, qc); }
        if (k < g.nc[2]) { int qc = cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2])); t += T.nd[qc] * V(p + sz, qc); }
        s += c * t;
    }
    return y - s;
}

// ---- streaming CG phases (vectors in global memory) --------------------------------
// Two nodes per loop trip with __restrict__ operands so both nodes' 14 stencil loads
// are in flight together (memory-level parallelism for the HBM-bound grids).

// phase A for one node: pp = z (+ beta p_old), qv = (A_c p)_p
__device__ __forceinline__ void stream_a_node(const Grid& g, const ClassTable& T, int p,
                                              const double* __restrict__ r, const double* __restrict__ pold,
                                              bool first, double beta, double& pp, double& qv) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    if (i >= 2 && i <= g.nc[0] - 2 && j >= 2 && j <= g.nc[1] - 2 && k >= 2 && k <= g.nc[2] - 2) {
        // node and neighbours interior: constant coefficients (class 13)
        const double ivc = T.invd[13];
        auto pc = [&](int q) -> double {
            const double z = __dmul_rn(ivc, r[q]);
            return first ? z : __dadd_rn(__dmul_rn(beta, pold[q]), z);
        };
        pp = pc(p);
        const double tx_ = pc(p - 1) + pc(p + 1);
        const double ty_ = pc(p - sy) + pc(p + sy);
        const double tz_ = pc(p - sz) + pc(p + sz);
        qv = T.diag[13] * pp - ((T.c[0][13] * tx_ + T.c[1][13] * ty_) + T.c[2][13] * tz_);
    } else {
        const int cls = class_of(g, i, j, k);
        auto pn = [&](int q, int qc) -> double {
            const double z = __dmul_rn(T.invd[qc], r[q]);
            return first ? z : __dadd_rn(__dmul_rn(beta, pold[q]), z);
        };
        pp = pn(p, cls);
        qv = (T.nd[cls] == 0.0) ? pp : apply_free(g, T, p, i, j, k, cls, pp, pn);
    }
}

// L2 prefetch of the lines a sweep will first touch kPfTrips grid-stride trips ahead
// (the +z plane of the stencil vectors and the unit-stride vectors): raises the DRAM
// requests in flight without holding registers.
constexpr int kPfTrips = 4;

__device__ __forceinline__ void prefetch_l2(const double* a) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// Nodes beg, beg+stride, ... < end; lim bounds the stored index range (prefetch only).
__device__ __forceinline__ double stream_phase_a(const Grid& g, const ClassTable& T, int beg, int stride,
                                                 int end, int lim, const double* __restrict__ r,
                                                 const double* __restrict__ pold, double* __restrict__ pnew,
                                                 bool first, double beta) {
    double pq = 0.0;
    int p = beg;
    const int sz = g.NX * g.NY;
    for (; p + stride < end; p += 2 * stride) {
        const int pf = p + kPfTrips * stride + sz;
        if (pf < lim) {
            prefetch_l2(r + pf);
            if (!first) prefetch_l2(pold + pf);
        }
        double pa, qa, pb, qb;
        stream_a_node(g, T, p, r, pold, first, beta, pa, qa);
        stream_a_node(g, T, p + stride, r, pold, first, beta, pb, qb);
        pnew[p] = pa;
        pnew[p + stride] = pb;
        pq += pa * qa;
        pq += pb * qb;
    }
    if (p < end) {
        double pa, qa;
        stream_a_node(g, T, p, r, pold, first, beta, pa, qa);
        pnew[p] = pa;
        pq += pa * qa;
    }
    return pq;
}

// phase B for one node: q recomputed from the stored p; returns (x_new, r_new, invd)
__device__ __forceinline__ void stream_b_node(const Grid& g, const ClassTable& T, int p,
                                              const double* __restrict__ pnew, double& pp, double& qv,
                                              double& iv) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int cls = class_of(g, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    pp = pnew[p];
    iv = T.invd[cls];
    if (i >= 1 && i <= g.nc[0] - 1 && j >= 1 && j <= g.nc[1] - 1 && k >= 2 && k <= g.nc[2] - 1 &&
        (g.dkind != kGamma || (i >= 2 && i <= g.nc[0] - 2 && j >= 2 && j <= g.nc[1] - 2))) {
        // interior class with six free neighbours
        qv = T.diag[13] * pp - ((T.c[0][13] * (pnew[p - 1] + pnew[p + 1]) +
                                 T.c[1][13] * (pnew[p - sy] + pnew[p + sy])) +
                                T.c[2][13] * (pnew[p - sz] + pnew[p + sz]));
    } else {
        qv = (T.nd[cls] == 0.0) ? pp : apply_free(g, T, p, i, j, k, cls, pp, [&](int q, int) { return pnew[q]; });
    }
}

__device__ __forceinline__ void stream_phase_b(const Grid& g, const ClassTable& T, int beg, int stride,
                                               int end, int lim, double* __restrict__ x, double* __restrict__ r,
                                               const double* __restrict__ pnew, double alpha, double& rz,
                                               double& rr) {
    auto finish = [&](int p, double pp, double qv, double iv) {
        const double xv = __dadd_rn(x[p], __dmul_rn(alpha, pp));
        const double rv = __dsub_rn(r[p], __dmul_rn(alpha, qv));
        x[p] = xv;
        r[p] = rv;
        const double z = __dmul_rn(iv, rv);
        rz += rv * z;
        rr += rv * rv;
    };
    int p = beg;
    const int sz = g.NX * g.NY;
    for (; p + stride < end; p += 2 * stride) {
        const int pf = p + kPfTrips * stride;
        if (pf + sz < lim) prefetch_l2(pnew + pf + sz);
        if (pf < end) {
            prefetch_l2(x + pf);
            prefetch_l2(r + pf);
        }
        double pa, qa, ia, pb, qb, ib;
        stream_b_node(g, T, p, pnew, pa, qa, ia);
        stream_b_node(g, T, p + stride, pnew, pb, qb, ib);
        finish(p, pa, qa, ia);
        finish(p + stride, pb, qb, ib);
    }
    if (p < end) {
        double pa, qa, ia;
        stream_b_node(g, T, p, pnew, pa, qa, ia);
        finish(p, pa, qa, ia);
    }
}

// ---------------------------------------------------------------------------------
// Persistent cooperative PCG.  grid.sync() separates the phases:
//   phase 0: b, r = b, x = 0, partial ||b||^2 and r.z             | sync
//   loop:    test ||r|| < rtol ||b||  (scipy: top of each iteration)
//            phase A: p = z (first) or beta p + z; q = A_c p; p.q | sync
//            phase B: x += alpha p; r -= alpha q; r.z, r.r        | sync
//   final:   ||A_c x - b||, non-finite check                      | sync
//            x_D = g, info
// ---------------------------------------------------------------------------------
template <bool GAUSS>
__global__ void __launch_bounds__(kTPB, 2) k_pcg(PcgParams P) {
    cg::grid_group grid = cg::this_grid();
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    __shared__ double tot[4];
    extern __shared__ double gtab[];
    const Grid& g = P.g;
    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    double *tx = gtab, *ty = gtab + 6 * g.nc[0], *tz = ty + 6 * g.nc[1];
    double *bx_ = tz + 6 * g.nc[2], *by_ = bx_ + g.NX, *bz_ = by_ + g.NY;
    if (GAUSS) build_gauss_tables(g, P.src, tx, ty, tz);
    __syncthreads();
    if (GAUSS) {
        build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
        __syncthreads();
    }

    const int G = gridDim.x;
    // nodes interleaved across CTAs (grid stride): faces and edges, which take the
    // class-table path, are spread evenly instead of landing on a few CTAs
    const int beg = blockIdx.x * kTPB + threadIdx.x;
    const int stride = G * kTPB;
    const int end = g.n;

    // ---- phase 0: constrained RHS (fem.py:169-191 + 89-105) ----
    double acc[2] = {0.0, 0.0};
    for (int p = beg; p < end; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        const int cls = class_of(g, i, j, k);
        double bv;
        if (T.nd[cls] == 0.0) {
            bv = dirichlet_value(P, p);
        } else {
            bv = T.mass[cls] * P.T[p];
            if (P.load) bv += P.load[p];
            if (GAUSS) bv = add_gaussian(bv, g, tx, ty, tz, bx_, by_, bz_, i, j, k);
            bv += dirichlet_lift(P, T, p, i, j, k, cls);
        }
        P.b[p] = bv;
        P.r[p] = bv;
        P.T[p] = 0.0;
        const double z = __dmul_rn(T.invd[cls], bv);
        acc[0] += bv * bv;
        acc[1] += bv * z;
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) { P.part[0 * G + blockIdx.x] = acc[0]; P.part[1 * G + blockIdx.x] = acc[1]; }
    grid.sync();
    {
        const int s[2] = {0, 1};
        grid_sum_fast<2, kResMaxBlocks>(P.part, s, G, tot);
    }
    const double bb = tot[0];
    double rz = tot[1];
    const double bnorm = sqrt(bb);
    const double atol = P.rtol * bnorm;
    double rnorm = bnorm;
    int it = 0, status = 0;
    double rho_prev = 1.0;
    double* pold = P.p0;
    double* pnew = P.p1;

    if (bb == 0.0) {
        status = 0;   // fem.py:275-276: zero solution
    } else {
        while (true) {
            // scipy's cg: `for it in range(maxiter): if ||r|| < atol: return ok`, failure when
            // the loop runs out -- the limit is tested before the residual
            if (it >= P.maxiter) { status = 1; break; }
            if (rnorm < atol) { status = 0; break; }
            if (!isfinite(rnorm)) { status = 3; break; }
            const double rho = rz;
            const double beta = it > 0 ? rho / rho_prev : 0.0;
            const bool first = it == 0;
            // ---- phase A: p = z (+ beta p), q = A_c p only for p.q (q is recomputed in B,
            //      so each iteration moves 64 B/node: r, p read + p written here, x, r, p
            //      read + x, r written in B).  Nodes two or more away from every face
            //      take the constant-coefficient path (their neighbours are interior too). ----
            double pq[1] = {stream_phase_a(g, T, beg, stride, g.n, g.n, P.r, pold, pnew, first, beta)};
            block_sum<1>(pq, red);
            if (threadIdx.x == 0) P.part[2 * G + blockIdx.x] = pq[0];
            grid.sync();
            {
                const int s[1] = {2};
                grid_sum_fast<1, kResMaxBlocks>(P.part, s, G, tot);
            }
            const double alpha = rho / tot[0];
            // ---- phase B ----
            double a2[2] = {0.0, 0.0};
            stream_phase_b(g, T, beg, stride, g.n, g.n, P.T, P.r, pnew, alpha, a2[0], a2[1]);
            block_sum<2>(a2, red);
            if (threadIdx.x == 0) { P.part[0 * G + blockIdx.x] = a2[0]; P.part[1 * G + blockIdx.x] = a2[1]; }
            grid.sync();
            {
                const int s[2] = {0, 1};
                grid_sum_fast<2, kResMaxBlocks>(P.part, s, G, tot);
            }
            rz = tot[0];
            rnorm = sqrt(tot[1]);
            rho_prev = rho;
            double* t = pold; pold = pnew; pnew = t;
            ++it;
        }
    }

    // ---- true residual ||A_c x - b|| / ||b|| (fem.py:286) and finite check ----
    double res[2] = {0.0, 0.0};
    for (int p = beg; p < end; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        const int cls = class_of(g, i, j, k);
        const double xp = P.T[p];
        double ax;
        if (T.nd[cls] == 0.0) ax = xp;
        else ax = apply_free(g, T, p, i, j, k, cls, xp, [&](int q, int) { return P.T[q]; });
        const double d = ax - P.b[p];
        res[0] += d * d;
        res[1] += isfinite(xp) ? 0.0 : 1.0;
    }
    block_sum<2>(res, red);
    if (threadIdx.x == 0) { P.part[0 * G + blockIdx.x] = res[0]; P.part[3 * G + blockIdx.x] = res[1]; }
    grid.sync();
    {
        const int s[2] = {0, 3};
        grid_sum_fast<2, kResMaxBlocks>(P.part, s, G, tot);
    }
    const double tres = bnorm > 0.0 ? sqrt(tot[0]) / bnorm : 0.0;
    // ---- re-impose Dirichlet values (fem.py:289-290): x_D = g = b_D ----
    for (int p = beg; p < end; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        const int cls = class_of(g, i, j, k);
        if (T.nd[cls] == 0.0) P.T[p] = P.b[p];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (status == 0 && tot[1] > 0.0) status = 3;
        if (status == 0 && (!isfinite(tres) || tres > 1e2 * P.rtol)) status = 2;
        P.info->iterations = (status == 1) ? P.maxiter : it;
        P.info->status = status;
        P.info->bnorm = bnorm;
        P.info->rnorm = rnorm;
        P.info->true_resid = tres;
    }
}

// ---------------------------------------------------------------------------------
// Gaussian nodal load as a dense array, for the streaming solve (keeps the Gaussian's
// registers out of the iteration loop).  Applies the same exact cutoff as add_gaussian
// against b0 = (rho c/dt) V n_p/24 * T_old: load = F, or 0 where F cannot change b0.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gauss_load(Grid g, Gauss src, double mbase, const double* T,
                                                    double* load) {
    extern __shared__ double gtab[];
    __shared__ double massc[27];
    double *tx = gtab, *ty = tx + 6 * g.nc[0], *tz = ty + 6 * g.nc[1];
    double *bx_ = tz + 6 * g.nc[2], *by_ = bx_ + g.NX, *bz_ = by_ + g.NY;
    build_gauss_tables(g, src, tx, ty, tz);
    if (threadIdx.x < 27) {
        int n_p, n_e[3], cnt[3], h0[3], h1[3];
        class_counts(threadIdx.x, n_p, n_e, cnt, h0, h1);
        massc[threadIdx.x] = class_is_dirichlet(threadIdx.x, g.dkind) ? -1.0 : mbase * (double)n_p;
    }
    __syncthreads();
    build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
    __syncthreads();
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
        int i, j, k;
        decode(g, p, i, j, k);
        const double m = massc[class_of(g, i, j, k)];
        if (m < 0.0) { load[p] = 0.0; continue; }
        const double b0 = m * T[p];
        const double bound = 24.0 * bx_[i] * by_[j] * bz_[k];
        load[p] = (b0 > 0.0 && bound < b0 * 0x1p-55) ? 0.0 : gaussian_node_fast(g, tx, ty, tz, i, j, k);
    }
}

// ---------------------------------------------------------------------------------
// Kuhn-P1 location in a grid (mesh.py:308-339; the grid may be a translated local one): cell
// by floor((x-lo)/h) clipped; tet by the descending order of the in-cell fractions.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double p1_eval(const Grid& G, const double* v, double x, double y, double z) {
    const double pt[3] = {x, y, z};
    int c[3];
    double xi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int ci = (int)floor((pt[a] - (G.lo0[a] + G.off[a])) / G.h[a]);      // the grid may be translated
        ci = ci < 0 ? 0 : (ci > G.nc[a] - 1 ? G.nc[a] - 1 : ci);
        c[a] = ci;
        xi[a] = (pt[a] - node_coord(G, a, ci)) / G.h[a];
    }
    // sort axes by xi descending (stable on ties)
    int o0 = 0, o1 = 1, o2 = 2;
    if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
    if (xi[o2] > xi[o1]) { int t = o1; o1 = o2; o2 = t; }
    if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
    const int st[3] = {1, G.NX, G.NX * G.NY};
    const int n0 = c[0] + G.NX * (c[1] + G.NY * c[2]);
    const int n1 = n0 + st[o0];
    const int n2 = n1 + st[o1];
    const int n3 = n2 + st[o2];
    const double w0 = 1.0 - xi[o0], w1 = xi[o0] - xi[o1], w2 = xi[o1] - xi[o2], w3 = xi[o2];
    return w0 * v[n0] + w1 * v[n1] + w2 * v[n2] + w3 * v[n3];
}

// Kuhn-P1 location (Mesh.locate, mesh.py:308-339): the 4 vertex ids and barycentrics
// of the global tet holding (x, y, z); the same cell/tet choice as p1_eval.
__device__ __forceinline__ void p1_locate(const Grid& G, double x, double y, double z, int (&nd)[4],
                                          double (&w)[4]) {
    const double pt[3] = {x, y, z};
    int c[3];
    double xi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int ci = (int)floor((pt[a] - (G.lo0[a] + G.off[a])) / G.h[a]);      // the grid may be translated
        ci = ci < 0 ? 0 : (ci > G.nc[a] - 1 ? G.nc[a] - 1 : ci);
        c[a] = ci;
        xi[a] = (pt[a] - node_coord(G, a, ci)) / G.h[a];
    }
    int o0 = 0, o1 = 1, o2 = 2;
    if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
    if (xi[o2] > xi[o1]) { int t = o1; o1 = o2; o2 = t; }
    if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
    const int st[3] = {1, G.NX, G.NX * G.NY};
    nd[0] = c[0] + G.NX * (c[1] + G.NY * c[2]);
    nd[1] = nd[0] + st[o0];
    nd[2] = nd[1] + st[o1];
    nd[3] = nd[2] + st[o2];
    w[0] = 1.0 - xi[o0];
    w[1] = xi[o0] - xi[o1];
    w[2] = xi[o1] - xi[o2];
    w[3] = xi[o2];
}

// Interface facets of the local grid (extract_interface, mesh.py:477-523: LATERAL +
// BOTTOM): faces (x lo, x hi, y lo, y hi, z lo); per face cell (jb inner, jc outer) two
// triangles, each the face of one Kuhn tet; 3 edge-midpoint quadrature points of weight
// area/3 (mesh.py:131-137).  Low side of axis a: tets stepping a last, perm (b,c,a) /
// (c,b,a), facet (v0,v1,v2), dT/dn = -(T(v3) - T(v2)) / h_a.  High side: tets stepping a
// first, perm (a,b,c) / (a,c,b), facet (v1,v2,v3), dT/dn = (T(v1) - T(v0)) / h_a.
// Entry e = 3 f + q writes 4 (global node, density * barycentric) pairs at 4 e + r.
// np.interp over a (T, value) table: clamped outside, linear inside (materials.py:91-100)
struct KTab {
    const double* T;
    const double* v;
    int n;            // 0: no table
};

__device__ __forceinline__ double tab_interp(double x, const double* xp, const double* fp, int n) {
    if (!(x > xp[0])) return fp[0];
    if (!(x < xp[n - 1])) return fp[n - 1];
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xp[mid] <= x) lo = mid; else hi = mid;
    }
    const double slope = (fp[lo + 1] - fp[lo]) / (xp[lo + 1] - xp[lo]);
    return slope * (x - xp[lo]) + fp[lo];
}

// jump = kappa_global(T_qp) - kappa_local(T_qp) when both tables are given (T_qp: the
// local P1 value at the quadrature point, the edge midpoint average), else the constant.
__global__ void k_trans_entries(Grid G, Grid L, const double* __restrict__ T, double jump, KTab kg, KTab kl,
                                int nfacet, int* __restrict__ keys, int* __restrict__ idx,
                                double* __restrict__ vals) {
    const int faceA[5] = {0, 0, 1, 1, 2}, faceS[5] = {0, 1, 0, 1, 0};
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 3 * nfacet; e += gridDim.x * blockDim.x) {
        int f = e / 3;
        const int q = e - 3 * f;
        int fi = 0, a = 0, side = 0, b = 0, c = 0, cnt = 0;
        for (fi = 0; fi < 5; ++fi) {
            a = faceA[fi];
            side = faceS[fi];
            b = a == 0 ? 1 : 0;
            c = a == 2 ? 1 : 2;
            cnt = 2 * L.nc[b] * L.nc[c];
            if (f < cnt) break;
            f -= cnt;
        }
        const int t = f & 1;
        const int jb = (f >> 1) % L.nc[b], jc = (f >> 1) / L.nc[b];
        int cell[3];
        cell[a] = side == 0 ? 0 : L.nc[a] - 1;
        cell[b] = jb;
        cell[c] = jc;
        int perm[3];
        if (side == 0) { perm[0] = t == 0 ? b : c; perm[1] = t == 0 ? c : b; perm[2] = a; }
        else { perm[0] = a; perm[1] = t == 0 ? b : c; perm[2] = t == 0 ? c : b; }
        int v[4][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) v[0][d] = cell[d];
#pragma unroll
        for (int r = 1; r < 4; ++r) {
#pragma unroll
            for (int d = 0; d < 3; ++d) v[r][d] = v[r - 1][d];
            v[r][perm[r - 1]] += 1;
        }
        auto nid = [&](const int* u) { return u[0] + L.NX * (u[1] + L.NY * u[2]); };
        double dTdn;
        int tri0;
        if (side == 0) {
            dTdn = -(T[nid(v[3])] - T[nid(v[2])]) / L.h[a];
            tri0 = 0;
        } else {
            dTdn = (T[nid(v[1])] - T[nid(v[0])]) / L.h[a];
            tri0 = 1;
        }
        const int pa = q == 2 ? 0 : q, pb = q == 0 ? 1 : 2;      // edges (0,1) (1,2) (0,2)
        const int* A = v[tri0 + pa];
        const int* B = v[tri0 + pb];
        double x[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) x[d] = 0.5 * (node_coord(L, d, A[d]) + node_coord(L, d, B[d]));
        double jq = jump;
        if (kg.n > 0) {
            const double tq = 0.5 * (T[nid(A)] + T[nid(B)]);
            jq = tab_interp(tq, kg.T, kg.v, kg.n) - tab_interp(tq, kl.T, kl.v, kl.n);
        }
        const double dens = 0.5 * L.h[b] * L.h[c] / 3.0 * jq * dTdn;
        int nd[4];
        double w[4];
        p1_locate(G, x[0], x[1], x[2], nd, w);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            keys[4 * e + r] = nd[r];
            idx[4 * e + r] = 4 * e + r;
            vals[4 * e + r] = dens * w[r];
        }
    }
}

// Ordered segment sums over the key-sorted entries (stable sort: entry order within a
// node) -> load[node]; deterministic, no atomics.
__global__ void k_trans_segsum(const int* __restrict__ skeys, const int* __restrict__ sidx,
                               const double* __restrict__ vals, int ne, double* __restrict__ load) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ne; j += gridDim.x * blockDim.x) {
        const int key = skeys[j];
        if (j > 0 && skeys[j - 1] == key) continue;
        double s = 0.0;
        for (int u = j; u < ne && skeys[u] == key; ++u) s += vals[sidx[u]];
        load[key] = s;
    }
}

// mode 0: all target nodes -> out_all (and gamma nodes also -> out_gamma if non-null)
// mode 1: gamma nodes only -> out_gamma
__global__ void k_interp(Grid G, const double* __restrict__ v, Grid L, int mode, double* out_all,
                         double* out_gamma) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L.n; p += gridDim.x * blockDim.x) {
        int i, j, k;
        decode(L, p, i, j, k);
        const bool gam = (k == 0) || i == 0 || i == L.nc[0] || j == 0 || j == L.nc[1];
        if (mode == 1 && !gam) continue;
        const double val = p1_eval(G, v, node_coord(L, 0, i), node_coord(L, 1, j), node_coord(L, 2, k));
        if (mode == 0) out_all[p] = val;
        if (gam && out_gamma) out_gamma[p] = val;
    }
}

__global__ void k_interp_pts(Grid G, const double* __restrict__ v, const double* __restrict__ pts,
                             int64_t np, double* out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < np; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = p1_eval(G, v, pts[3 * e], pts[3 * e + 1], pts[3 * e + 2]);
}

// ---------------------------------------------------------------------------------
// Deposit: one block.  Zero the nodes written last call, then scatter the new
// samples with barycentric weights and merge repeated nodes in sample order
// (np.add.at order), writing load[node] = sum.
// ---------------------------------------------------------------------------------
constexpr int kDepMax = 2048;   // contributions per call (samples * 4)

// Only nodes in [lo, hi) are written (a slab's own nodes; 0..n for the whole grid);
// load may be base-shifted so that load[id] addresses global node id.
__global__ void __launch_bounds__(1024) k_deposit(Grid G, const double* __restrict__ pts,
                                                 const double* __restrict__ pw, int count,
                                                 double* load, int* prev_nodes, int* prev_count,
                                                 int lo, int hi) {
    __shared__ int s_node[kDepMax];
    __shared__ double s_val[kDepMax];
    const int np = *prev_count;
    for (int e = threadIdx.x; e < np; e += blockDim.x) load[prev_nodes[e]] = 0.0;
    __syncthreads();
    const int nc = min(count * 4, kDepMax);
    for (int s = threadIdx.x; s < count && s * 4 < kDepMax; s += blockDim.x) {
        const double pt[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
        int c[3];
        double xi[3];
        for (int a = 0; a < 3; ++a) {
            int ci = (int)floor((pt[a] - (G.lo0[a] + G.off[a])) / G.h[a]);      // the grid may be translated
            ci = ci < 0 ? 0 : (ci > G.nc[a] - 1 ? G.nc[a] - 1 : ci);
            c[a] = ci;
            xi[a] = (pt[a] - node_coord(G, a, ci)) / G.h[a];
        }
        int o0 = 0, o1 = 1, o2 = 2;
        if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
        if (xi[o2] > xi[o1]) { int t = o1; o1 = o2; o2 = t; }
        if (xi[o1] > xi[o0]) { int t = o0; o0 = o1; o1 = t; }
        const int st[3] = {1, G.NX, G.NX * G.NY};
        const int n0 = c[0] + G.NX * (c[1] + G.NY * c[2]);
        s_node[4 * s + 0] = n0;
        s_node[4 * s + 1] = n0 + st[o0];
        s_node[4 * s + 2] = n0 + st[o0] + st[o1];
        s_node[4 * s + 3] = n0 + st[o0] + st[o1] + st[o2];
        const double P = pw[s];
        s_val[4 * s + 0] = P * (1.0 - xi[o0]);
        s_val[4 * s + 1] = P * (xi[o0] - xi[o1]);
        s_val[4 * s + 2] = P * (xi[o1] - xi[o2]);
        s_val[4 * s + 3] = P * xi[o2];
    }
    __syncthreads();
    // first occurrences write the in-order sum
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nc; e += blockDim.x) {
        const int nd = s_node[e];
        bool first = true;
        for (int f = 0; f < e; ++f)
            if (s_node[f] == nd) { first = false; break; }
        if (!first || nd < lo || nd >= hi) continue;
        double sum = 0.0;
        for (int f = e; f < nc; ++f)
            if (s_node[f] == nd) sum += s_val[f];
        load[nd] = sum;
        const int slot = atomicAdd(&s_cnt, 1);
        prev_nodes[slot] = nd;
    }
    __syncthreads();
    if (threadIdx.x == 0) *prev_count = s_cnt;
}

// max and count(T > T_l) of a field: per-block partials, finished by block 0 of a
// second launch (deterministic).
__global__ void k_melt_partial(const double* __restrict__ v, int n, double Tl, double* part) {
    __shared__ double smax[32], scnt[32];
    double m = -1e300, c = 0.0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const double t = v[p];
        m = fmax(m, t);
        c += t > Tl ? 1.0 : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { smax[wid] = m; scnt[wid] = c; }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        m = lane < nw ? smax[lane] : -1e300;
        c = lane < nw ? scnt[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) { part[2 * blockIdx.x] = m; part[2 * blockIdx.x + 1] = c; }
    }
}

__global__ void k_melt_final(const double* part, int nb, double* out_max, double* out_cnt) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double m = -1e300, c = 0.0;
        for (int b = 0; b < nb; ++b) { m = fmax(m, part[2 * b]); c += part[2 * b + 1]; }
        *out_max = m;
        *out_cnt = c;
    }
}

// v^T M v with the consistent P1 mass matrix of the Kuhn tets: per tet
// V/20 (sum v_i^2 + (sum v_i)^2), V = hx hy hz / 6 (the 4-point rule of the reference's
// mass_matrix is exact for P1 x P1).  One thread per cell gathers the 8 corners of
// d = a - b (d = a when b == nullptr) and of b; the six Kuhn tets of a cell share the
// main diagonal 000-111 and run 000 -> e_pi0 -> e_pi0 + e_pi1 -> 111.  Per-block partials
// (fixed order, deterministic) go to part[2 * block + {0, 1}].
__global__ void k_mass_norms(Grid L, const double* __restrict__ a, const double* __restrict__ b,
                             double* part) {
    __shared__ double red[64];
    const int ncell = L.nc[0] * L.nc[1] * L.nc[2];
    const int sy = L.NX, sz = L.NX * L.NY;
    double acc[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const int ci = c % L.nc[0], t = c / L.nc[0];
        const int cj = t % L.nc[1], ck = t / L.nc[1];
        const int p0 = ci + sy * cj + sz * ck;
        const int off[8] = {0, 1, sy, 1 + sy, sz, 1 + sz, sy + sz, 1 + sy + sz};   // bit a = axis a
        double d[8], r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double av = a[p0 + off[q]];
            const double bv = b ? b[p0 + off[q]] : 0.0;
            d[q] = b ? av - bv : av;
            r[q] = bv;
        }
        double sd = 0.0, sr = 0.0;
        // permutations in itertools order: (0,1,2) (0,2,1) (1,0,2) (1,2,0) (2,0,1) (2,1,0)
        const int mid[6][2] = {{1, 3}, {1, 5}, {2, 3}, {2, 6}, {4, 5}, {4, 6}};
#pragma unroll
        for (int e = 0; e < 6; ++e) {
            const int v1 = mid[e][0], v2 = mid[e][1];
            const double s1 = d[0] + d[v1] + d[v2] + d[7];
            sd += d[0] * d[0] + d[v1] * d[v1] + d[v2] * d[v2] + d[7] * d[7] + s1 * s1;
            const double s2 = r[0] + r[v1] + r[v2] + r[7];
            sr += r[0] * r[0] + r[v1] * r[v1] + r[v2] * r[v2] + r[7] * r[7] + s2 * s2;
        }
        acc[0] += sd;
        acc[1] += sr;
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        const double w = L.h[0] * L.h[1] * L.h[2] / 6.0 / 20.0;
        part[2 * blockIdx.x] = acc[0] * w;
        part[2 * blockIdx.x + 1] = acc[1] * w;
    }
}

// Masked mass norms (twolevel.masked_mass, twolevel.py:361-373): (a-b)^T M (a-b) over the
// tets whose centroid lies in the closed box [blo, bhi] -> part[2 blk], the others ->
// part[2 blk + 1] (consistency_diagnostic's overlap / exterior split, :376-400).
__global__ void k_mass_norms_split(Grid L, const double* __restrict__ a, const double* __restrict__ b,
                                   double blo0, double blo1, double blo2, double bhi0, double bhi1, double bhi2,
                                   double* part) {
    __shared__ double red[64];
    const int ncell = L.nc[0] * L.nc[1] * L.nc[2];
    const int sy = L.NX, sz = L.NX * L.NY;
    const double blo[3] = {blo0, blo1, blo2}, bhi[3] = {bhi0, bhi1, bhi2};
    double acc[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const int ci = c % L.nc[0], t = c / L.nc[0];
        const int cj = t % L.nc[1], ck = t / L.nc[1];
        const int cc[3] = {ci, cj, ck};
        const int p0 = ci + sy * cj + sz * ck;
        const int off[8] = {0, 1, sy, 1 + sy, sz, 1 + sz, sy + sz, 1 + sy + sz};
        double d[8];
        for (int q = 0; q < 8; ++q) d[q] = a[p0 + off[q]] - b[p0 + off[q]];
        const int mid[6][2] = {{1, 3}, {1, 5}, {2, 3}, {2, 6}, {4, 5}, {4, 6}};
        for (int e = 0; e < 6; ++e) {
            const int v[4] = {0, mid[e][0], mid[e][1], 7};
            bool in = true;
            for (int ax = 0; ax < 3; ++ax) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += node_coord(L, ax, cc[ax] + ((v[k] >> ax) & 1));
                const double cen = s / 4.0;
                in = in && cen >= blo[ax] && cen <= bhi[ax];
            }
            const double s1 = d[0] + d[v[1]] + d[v[2]] + d[7];
            const double f = d[0] * d[0] + d[v[1]] * d[v[1]] + d[v[2]] * d[v[2]] + d[7] * d[7] + s1 * s1;
            acc[in ? 0 : 1] += f;
        }
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        const double w = L.h[0] * L.h[1] * L.h[2] / 6.0 / 20.0;
        part[2 * blockIdx.x] = acc[0] * w;
        part[2 * blockIdx.x + 1] = acc[1] * w;
    }
}

__global__ void k_flush(double* buf, size_t n, double v) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
        buf[e] = v;
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int n) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) b[e] = a[e];
}

// dst[e] = src[idx[e]] (the trace entries of a dense local array: tl_run_get_field_at)
__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ idx, int n, double* __restrict__ dst) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) dst[e] = src[idx[e]];
}

// The values k_interp writes at the listed target nodes (same arithmetic: bitwise equal).
__global__ void k_interp_nodes(Grid G, const double* __restrict__ v, Grid L, const int* __restrict__ idx, int n,
                               double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        int i, j, k;
        const int p = idx[e];
        if (p < 0 || p >= L.n) { out[e] = nan(""); continue; }     // not a node of the target lattice
        decode(L, p, i, j, k);
        out[e] = p1_eval(G, v, node_coord(L, 0, i), node_coord(L, 1, j), node_coord(L, 2, k));
    }
}

__global__ void k_axpy(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
        y[e] = __dadd_rn(__dmul_rn(a, x[e]), y[e]);
}

// Dirichlet data given as a node list: mask and values of a dense pair (cleared before)
__global__ void k_scatter_dirichlet(const int* __restrict__ nodes, const double* __restrict__ vals, int nd, int n,
                                    unsigned char* __restrict__ mask, double* __restrict__ g) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nd; e += gridDim.x * blockDim.x) {
        const int p = nodes[e];
        if (p >= 0 && p < n) {
            if (mask) mask[p] = 1;
            g[p] = vals[e];
        }
    }
}

__global__ void k_fill(double* a, int n, double v) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) a[e] = v;
}

}  // namespace tl
