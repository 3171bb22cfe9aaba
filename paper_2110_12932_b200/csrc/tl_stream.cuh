// tl_stream.cuh — streaming Jacobi-PCG for grids that do not fit on chip (sm_100a, fp64).
//
// Same operator, RHS, stopping rule and final checks as k_pcg / scipy's cg
// (lpbfsim/fem.py:129-194, 89-105, 271-298), split into four launches so that the CG
// loop kernel holds only the two sweeps and runs at 3 x 512 threads per SM (40 registers;
// the memory-level parallelism an HBM-bound sweep needs):
//
//   k_s_rhs    constrained RHS b, r = b, x = 0, block partials of ||b||^2 and r.z
//   k_s_cg     cooperative CG loop: sweep A | grid sync | sweep B | grid sync
//   k_s_resid  ||A_c x - b|| and non-finite partials (fem.py:286), then x_D = g (:289-290)
//   k_s_final  one block sums the residual partials -> info
//
// Sweep A forms p = z + beta p_old and the alpha denominator p.Ap.  Instead of
// recomputing p at all seven stencil points (14 loads per node), p.Ap is summed over the
// node and its three FORWARD edges:
//     p.Ap = sum_p d_p p_p^2 - 2 sum_{edges (p, p+e_a), both free} c_a p_p p_{p+e_a}
// (A is symmetric after the symmetric Dirichlet elimination and c_a depends only on the
// edge; identity rows contribute p_p^2), so a node reads r and p_old at four points.
// Sweep B recomputes q = A p from the stored p (7-point) and updates x and r.  Per
// iteration the two sweeps move the algorithmic 64 B/node: 24 in A (r, p_old read, p
// written), 40 in B (p, x, r read, x, r written); neighbour reads hit L1/L2.
// Partial sums are reduced in a fixed order (deterministic; every CTA bitwise equal).
//
// Measured alternatives (profiles/README.md): a 2.5D z-march staging planes in shared
// memory with cp.async, and the same sweeps as plain kernels inside a CUDA graph with a
// device-side while node (cudaGraphSetConditional), were both slower on B200.
#pragma once

#include "tl_kernels.cuh"

namespace tl {

constexpr int kSTPB = 512;                 // threads per CTA of the streaming kernels
constexpr int kSMaxBlocks = 4 * kSTPB;     // grid_sum_wide capacity
constexpr int kSPartCG = 4096;             // offset of k_s_cg's partials in PcgParams::part

// Fixed-order sum of G <= 4 blockDim.x partials by the whole CTA in one L2 round trip:
// thread t adds partials t, t + B, t + 2B, t + 3B in that order, then the deterministic
// block_sum; every CTA computes bitwise the same totals (broadcast in smem_out).
template <int NV>
__device__ __forceinline__ void grid_sum_wide(const double* part, const int (&slot)[NV], int G,
                                              double* red, double* smem_out) {
    const int B = blockDim.x;
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = threadIdx.x + u * B;
            v[u] = b < G ? __ldcg(part + slot[k] * G + b) : 0.0;
        }
        s[k] = ((v[0] + v[1]) + v[2]) + v[3];
    }
    block_sum<NV>(s, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) smem_out[k] = s[k];
    __syncthreads();
}

// Node whose class is 13 and whose six neighbours are all free (sweep B's fast test): no
// Dirichlet lift, the constant-coefficient stencil.
__device__ __forceinline__ bool s_free_interior(const Grid& g, int i, int j, int k) {
    return i >= 1 && i <= g.nc[0] - 1 && j >= 1 && j <= g.nc[1] - 1 && k >= 2 && k <= g.nc[2] - 1 &&
           (g.dkind != kGamma || (i >= 2 && i <= g.nc[0] - 2 && j >= 2 && j <= g.nc[1] - 2));
}

// RHS value at node p = (i, j, k) from its T_old and dense-load values (fem.py:129-194 +
// constrained, 89-105); cls returns the node's class.
__device__ __forceinline__ double s_rhs_value(const PcgParams& P, const ClassTable& T, const int* box, int p, int i,
                                              int j, int k, double told, double loadv, int& cls) {
    const Grid& g = P.g;
    // the precomputed Gaussian load of the node (0 outside the box; Dirichlet nodes hold 0)
    auto boxload = [&]() -> double {
        if (i < box[0] || i >= box[1] || j < box[2] || j >= box[3] || k < box[4] || k >= box[5]) return 0.0;
        return P.bload[(i - box[0]) + (box[1] - box[0]) * ((j - box[2]) + (box[3] - box[2]) * (k - box[4]))];
    };
    double bv;
    cls = 13;
    if (s_free_interior(g, i, j, k)) {
        bv = T.mass[13] * told;
        if (P.load) bv += loadv;
        if (P.bload) bv += boxload();
    } else {
        cls = class_of(g, i, j, k);
        if (T.nd[cls] == 0.0) {
            bv = dirichlet_value(P, p);
        } else {
            bv = T.mass[cls] * told;
            if (P.load) bv += loadv;
            if (P.bload) bv += boxload();
            bv += dirichlet_lift(P, T, p, i, j, k, cls);
        }
    }
    return bv;
}

__device__ __forceinline__ double2 ld2(const double* a) { return *reinterpret_cast<const double2*>(a); }
__device__ __forceinline__ void st2(double* a, double v0, double v1) {
    *reinterpret_cast<double2*>(a) = make_double2(v0, v1);
}

// ---- k_s_rhs: b (and r = b, x = 0 unless the k_t_cg path implies them); partials
// [0][blk] = b.b, [1][blk] = r.z.  A thread takes the node pairs (2q, 2q + 1) of a grid-
// stride loop with 16-byte loads and stores (the arrays are 16-byte aligned and padded):
// half the memory instructions of a node-per-trip loop, twice the bytes in flight per thread.
__device__ __forceinline__ void s_rhs_block(const PcgParams& P) {
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    __shared__ int box[6];
    const Grid& g = P.g;
    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    if (threadIdx.x >= 32 && threadIdx.x < 38) box[threadIdx.x - 32] = P.bload ? P.bbox[threadIdx.x - 32] : 0;
    __syncthreads();
    double acc[2] = {0.0, 0.0};
    // (the dense load may sit at an odd offset of a workspace: 8-byte loads then)
    const bool lal = (reinterpret_cast<uintptr_t>(P.load) & 15) == 0;
    const int npair = g.n >> 1;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npair; q += gridDim.x * blockDim.x) {
        const int p = 2 * q;
        const double2 tv = ld2(P.T + p);
        const double2 lv = !P.load ? make_double2(0.0, 0.0)
                           : (lal ? ld2(P.load + p) : make_double2(P.load[p], P.load[p + 1]));
        int i, j, k, c0, c1;
        decode(g, p, i, j, k);
        const double b0 = s_rhs_value(P, T, box, p, i, j, k, tv.x, lv.x, c0);
        if (++i == g.NX) decode(g, p + 1, i, j, k);          // the pair straddles a row end
        const double b1 = s_rhs_value(P, T, box, p + 1, i, j, k, tv.y, lv.y, c1);
        st2(P.b + p, b0, b1);
        if (!P.light_rhs) {
            st2(P.r + p, b0, b1);
            st2(P.T + p, 0.0, 0.0);
        }
        acc[0] += b0 * b0;
        acc[1] += b0 * __dmul_rn(T.invd[c0], b0);
        acc[0] += b1 * b1;
        acc[1] += b1 * __dmul_rn(T.invd[c1], b1);
    }
    if ((g.n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {      // the odd last node
        const int p = g.n - 1;
        int i, j, k, c0;
        decode(g, p, i, j, k);
        const double b0 = s_rhs_value(P, T, box, p, i, j, k, P.T[p], P.load ? P.load[p] : 0.0, c0);
        P.b[p] = b0;
        if (!P.light_rhs) {
            P.r[p] = b0;
            P.T[p] = 0.0;
        }
        acc[0] += b0 * b0;
        acc[1] += b0 * __dmul_rn(T.invd[c0], b0);
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        P.part[blockIdx.x] = acc[0];
        P.part[gridDim.x + blockIdx.x] = acc[1];
    }
}

__global__ void __launch_bounds__(kSTPB, 3) k_s_rhs(PcgParams P) { s_rhs_block(P); }

// Batched (config 5): grid = (blocks per system, systems); system blockIdx.y from Ps.
__global__ void __launch_bounds__(kSTPB, 3) k_sb_rhs(const PcgParams* Ps) {
    __shared__ __align__(16) unsigned char pbuf[sizeof(PcgParams)];      // (PcgParams has default member initialisers)
    PcgParams& P = *reinterpret_cast<PcgParams*>(pbuf);
    for (int e = threadIdx.x; e < (int)(sizeof(PcgParams) / 4); e += blockDim.x)
        reinterpret_cast<uint32_t*>(pbuf)[e] = reinterpret_cast<const uint32_t*>(Ps + blockIdx.y)[e];
    __syncthreads();
    s_rhs_block(P);
}

// Sweep A at node p: p_p = z (+ beta p_old) written; returns p_p (A p)_p restricted to the
// node and its forward edges.
__device__ __forceinline__ double s_sweep_a_node(const Grid& g, const ClassTable& T, int p,
                                                 const double* __restrict__ r, const double* __restrict__ pold,
                                                 double* __restrict__ pnew, bool first, double beta) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    auto pv = [&](int q, double iv) -> double {
        const double z = __dmul_rn(iv, r[q]);
        return first ? z : __dadd_rn(__dmul_rn(beta, pold[q]), z);
    };
    double acc;
    if (i >= 1 && i <= g.nc[0] - 2 && j >= 1 && j <= g.nc[1] - 2 && k >= 1 && k <= g.nc[2] - 2) {
        // node and forward neighbours interior and free: class 13
        const double iv = T.invd[13];
        const double pp = pv(p, iv);
        pnew[p] = pp;
        const double px = pv(p + 1, iv), py = pv(p + sy, iv), pz = pv(p + sz, iv);
        acc = pp * (T.diag[13] * pp - 2.0 * ((T.c[0][13] * px + T.c[1][13] * py) + T.c[2][13] * pz));
    } else {
        const int cls = class_of(g, i, j, k);
        const double pp = pv(p, T.invd[cls]);
        pnew[p] = pp;
        if (T.nd[cls] == 0.0) {
            acc = pp * pp;                      // identity row
        } else {
            double t = 0.0;
            if (i < g.nc[0]) {
                const int qc = cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0]);
                if (T.nd[qc] != 0.0) t += T.c[0][cls] * pv(p + 1, T.invd[qc]);
            }
            if (j < g.nc[1]) {
                const int qc = cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1]));
                if (T.nd[qc] != 0.0) t += T.c[1][cls] * pv(p + sy, T.invd[qc]);
            }
            if (k < g.nc[2]) {
                const int qc = cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2]));
                if (T.nd[qc] != 0.0) t += T.c[2][cls] * pv(p + sz, T.invd[qc]);
            }
            acc = pp * (T.diag[cls] * pp - 2.0 * t);
        }
    }
    return acc;
}

// Sweep B at node p: q = A_c p from the stored p, x += alpha p, r -= alpha q; r.z, r.r.
__device__ __forceinline__ void s_sweep_b_node(const Grid& g, const ClassTable& T, int p, double* __restrict__ x,
                                               double* __restrict__ r, const double* __restrict__ pn,
                                               double alpha, double& rz, double& rr) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    const double pp = pn[p];
    double qv, iv;
    if (i >= 1 && i <= g.nc[0] - 1 && j >= 1 && j <= g.nc[1] - 1 && k >= 2 && k <= g.nc[2] - 1 &&
        (g.dkind != kGamma || (i >= 2 && i <= g.nc[0] - 2 && j >= 2 && j <= g.nc[1] - 2))) {
        iv = T.invd[13];
        qv = T.diag[13] * pp - ((T.c[0][13] * (pn[p - 1] + pn[p + 1]) + T.c[1][13] * (pn[p - sy] + pn[p + sy])) +
                                T.c[2][13] * (pn[p - sz] + pn[p + sz]));
    } else {
        const int cls = class_of(g, i, j, k);
        iv = T.invd[cls];
        qv = (T.nd[cls] == 0.0) ? pp : apply_free(g, T, p, i, j, k, cls, pp, [&](int q, int) { return pn[q]; });
    }
    const double xv = __dadd_rn(x[p], __dmul_rn(alpha, pp));
    const double rv = __dsub_rn(r[p], __dmul_rn(alpha, qv));
    x[p] = xv;
    r[p] = rv;
    rz += rv * __dmul_rn(iv, rv);
    rr += rv * rv;
}

// ---- k_s_cg: the CG iterations (cooperative).  Reads k_s_rhs's Grhs partials. ----------
template <int MINB, int UNR>
__global__ void __launch_bounds__(kSTPB, MINB) k_s_cg(PcgParams P, int Grhs) {
    cg::grid_group grid = cg::this_grid();
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    const Grid& g = P.g;
    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    {
        const int s[2] = {0, 1};
        grid_sum_wide<2>(P.part, s, Grhs, red, tot);   // also syncs T
    }
    const int G = gridDim.x;
    double* part = P.part + kSPartCG;
    const double bb = tot[0];
    double rz = tot[1];
    const double bnorm = sqrt(bb);
    const double atol = P.rtol * bnorm;
    double rnorm = bnorm;
    int it = 0, status = 0;
    double rho_prev = 1.0;
    double* pold = P.p0;
    double* pnew = P.p1;
    // CTA b takes the full 512-node chunks b, b + G, ...; the last CTA also the partial one
    const int stride = G * kSTPB;
    const int nfull = g.n / kSTPB, ptail = nfull * kSTPB + threadIdx.x;
    const bool tail = blockIdx.x == G - 1 && ptail < g.n;
    if (bb != 0.0) {
        while (true) {
            // scipy's cg: `for it in range(maxiter): if ||r|| < atol: return ok`, failure when
            // the loop runs out -- the limit is tested before the residual
            if (it >= P.maxiter) { status = 1; break; }
            if (rnorm < atol) { status = 0; break; }
            if (!isfinite(rnorm)) { status = 3; break; }
            const double rho = rz;
            const double beta = it > 0 ? rho / rho_prev : 0.0;
            const bool first = it == 0;
            unsigned long long* pf = (P.prof && it == 3 && threadIdx.x == 0 && blockIdx.x < 448)
                                         ? P.prof + 1024 + 16 * blockIdx.x : nullptr;
            if (pf) pf[0] = timer_ns();
            double pq[1] = {0.0};
            {
                int c = blockIdx.x;
                if (UNR == 2)
                    for (; c + G < nfull; c += 2 * G) {
                        const int p = c * kSTPB + threadIdx.x;
                        const double a = s_sweep_a_node(g, T, p, P.r, pold, pnew, first, beta);
                        const double b = s_sweep_a_node(g, T, p + stride, P.r, pold, pnew, first, beta);
                        pq[0] += a;
                        pq[0] += b;
                    }
                for (; c < nfull; c += G)
                    pq[0] += s_sweep_a_node(g, T, c * kSTPB + threadIdx.x, P.r, pold, pnew, first, beta);
                if (tail) pq[0] += s_sweep_a_node(g, T, ptail, P.r, pold, pnew, first, beta);
            }
            if (pf) pf[2] = timer_ns();
            block_sum<1>(pq, red);
            if (threadIdx.x == 0) part[blockIdx.x] = pq[0];
            grid.sync();
            if (pf) pf[3] = timer_ns();
            {
                const int s[1] = {0};
                grid_sum_wide<1>(part, s, G, red, tot);
            }
            if (pf) pf[4] = timer_ns();
            const double alpha = rho / tot[0];
            double a2[2] = {0.0, 0.0};
            {
                // snake: sweep B walks the 512-node chunks from the top of the grid down, so
                // it starts on the planes sweep A touched last (still in L2), and the next
                // sweep A starts where this one ends
                const int top = P.snake ? nfull - 1 : 0, sg = P.snake ? -1 : 1;
                int c = blockIdx.x;
                if (UNR == 2)
                    for (; c + G < nfull; c += 2 * G) {
                        const int p = (top + sg * c) * kSTPB + threadIdx.x;
                        s_sweep_b_node(g, T, p, P.T, P.r, pnew, alpha, a2[0], a2[1]);
                        s_sweep_b_node(g, T, p + sg * stride, P.T, P.r, pnew, alpha, a2[0], a2[1]);
                    }
                for (; c < nfull; c += G)
                    s_sweep_b_node(g, T, (top + sg * c) * kSTPB + threadIdx.x, P.T, P.r, pnew, alpha, a2[0], a2[1]);
                if (tail) s_sweep_b_node(g, T, ptail, P.T, P.r, pnew, alpha, a2[0], a2[1]);
            }
            if (pf) pf[6] = timer_ns();
            block_sum<2>(a2, red);
            if (threadIdx.x == 0) { part[G + blockIdx.x] = a2[0]; part[2 * G + blockIdx.x] = a2[1]; }
            grid.sync();
            if (pf) pf[7] = timer_ns();
            {
                const int s[2] = {1, 2};
                grid_sum_wide<2>(part, s, G, red, tot);
            }
            if (pf) pf[8] = timer_ns();
            rz = tot[0];
            rnorm = sqrt(tot[1]);
            rho_prev = rho;
            double* t = pold; pold = pnew; pnew = t;
            ++it;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.info->iterations = (status == 1) ? P.maxiter : it;
        P.info->status = status;
        P.info->bnorm = bnorm;
        P.info->rnorm = rnorm;
    }
}

// Residual term of node p: (A_c x - b)_p^2 and the non-finite count; then x_D = g = b_D
// (fem.py:289-290) after the node's own term (neighbours read x_D with weight nd = 0, so
// either value gives the same sum).
__device__ __forceinline__ void s_resid_node(const Grid& g, const ClassTable& T, int p, double* __restrict__ x,
                                             const double* __restrict__ b, double (&res)[2]) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    const double xp = x[p];
    const double bv = b[p];
    double ax;
    if (s_free_interior(g, i, j, k)) {
        ax = T.diag[13] * xp - ((T.c[0][13] * (x[p - 1] + x[p + 1]) + T.c[1][13] * (x[p - sy] + x[p + sy])) +
                                T.c[2][13] * (x[p - sz] + x[p + sz]));
    } else {
        const int cls = class_of(g, i, j, k);
        if (T.nd[cls] == 0.0) {
            ax = xp;
            x[p] = bv;
        } else {
            ax = apply_free(g, T, p, i, j, k, cls, xp, [&](int q, int) { return x[q]; });
        }
    }
    const double d = ax - bv;
    res[0] += d * d;
    res[1] += isfinite(xp) ? 0.0 : 1.0;
}

// ---- k_s_resid: partials [0][blk] = ||A_c x - b||^2, [1][blk] = non-finite count --------
__device__ __forceinline__ void s_resid_block(const PcgParams& P) {
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    const Grid& g = P.g;
    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    __syncthreads();
    double res[2] = {0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    for (; p + stride < g.n; p += 2 * stride) {
        s_resid_node(g, T, p, P.T, P.b, res);
        s_resid_node(g, T, p + stride, P.T, P.b, res);
    }
    if (p < g.n) s_resid_node(g, T, p, P.T, P.b, res);
    block_sum<2>(res, red);
    if (threadIdx.x == 0) {
        P.part[blockIdx.x] = res[0];
        P.part[gridDim.x + blockIdx.x] = res[1];
    }
}

__global__ void __launch_bounds__(kSTPB, 3) k_s_resid(PcgParams P) { s_resid_block(P); }

__global__ void __launch_bounds__(kSTPB, 3) k_sb_resid(const PcgParams* Ps) {
    __shared__ __align__(16) unsigned char pbuf[sizeof(PcgParams)];      // (PcgParams has default member initialisers)
    PcgParams& P = *reinterpret_cast<PcgParams*>(pbuf);
    for (int e = threadIdx.x; e < (int)(sizeof(PcgParams) / 4); e += blockDim.x)
        reinterpret_cast<uint32_t*>(pbuf)[e] = reinterpret_cast<const uint32_t*>(Ps + blockIdx.y)[e];
    __syncthreads();
    s_resid_block(P);
}

// ---- k_s_final (one block): the residual partials -> the outcome record ----------------
__device__ __forceinline__ void s_final_block(const PcgParams& P, int Gres) {
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    const int s[2] = {0, 1};
    grid_sum_wide<2>(P.part, s, Gres, red, tot);
    if (threadIdx.x == 0) {
        int status = P.info->status;
        const double bnorm = P.info->bnorm;
        const double tres = bnorm > 0.0 ? sqrt(tot[0]) / bnorm : 0.0;
        if (status == 0 && tot[1] > 0.0) status = 3;
        if (status == 0 && (!isfinite(tres) || tres > 1e2 * P.rtol)) status = 2;
        P.info->status = status;
        P.info->true_resid = tres;
    }
}

__global__ void __launch_bounds__(kSTPB) k_s_final(PcgParams P, int Gres) { s_final_block(P, Gres); }

__global__ void __launch_bounds__(kSTPB) k_sb_final(const PcgParams* Ps, int Gres) {
    __shared__ __align__(16) unsigned char pbuf[sizeof(PcgParams)];
    PcgParams& P = *reinterpret_cast<PcgParams*>(pbuf);
    for (int e = threadIdx.x; e < (int)(sizeof(PcgParams) / 4); e += blockDim.x)
        reinterpret_cast<uint32_t*>(pbuf)[e] = reinterpret_cast<const uint32_t*>(Ps + blockIdx.x)[e];
    __syncthreads();
    s_final_block(P, Gres);
}

}  // namespace tl
