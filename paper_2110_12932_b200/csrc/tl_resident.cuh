// tl_resident.cuh — SMEM-resident brick PCG for grids that fit on-chip (sm_100a, fp64).
//
// Same algorithm, operator and stopping rule as k_pcg (scipy cg mirrored, see
// tl_kernels.cuh), different data placement.  The grid is cut into one brick per
// SM.  Each CTA keeps its brick's p (with a one-node halo), r (with halo) and x in
// shared memory and q in registers for the whole solve; per iteration only the
// brick-surface values of r cross CTAs (written to a global exchange array before a
// grid barrier, read back into the neighbours' halos after it).  The halo p values
// are advanced by the same recurrence p = beta p + M^-1 r as their owners, so they
// stay bitwise identical without a second exchange.  Two grid barriers per
// iteration carry the two CG reductions (p.q, then r.z and r.r).
//
// Shared memory (per CTA, H = halo'd brick nodes, n = own nodes, F = halo face cells):
//   [Gaussian tables][PS: H doubles][RS: H][XS: n][GID: n ints][FS: F ints][FG: F ints][CL: H bytes]
#pragma once

#include "tl_kernels.cuh"

namespace tl {

constexpr int kResTPB = 512;
constexpr int kResMaxSplit = 64;
constexpr int kResKF = 8;              // halo face cells per thread (F <= kResKF * kResTPB)
constexpr uint8_t kNoNode = 27;

struct ResParams {
    PcgParams P;                  // grid, coefficients, inputs, workspace (b, part, info)
    double* xg;                   // global exchange array (brick-surface r), n doubles
    double* xx;                   // global exchange array (brick-surface x), n doubles
    unsigned long long* prof;     // optional phase timestamps (block 0), or nullptr
    int ng[3];                    // bricks per axis
    int off[3][kResMaxSplit + 1]; // brick boundaries per axis (node indices)
};

__host__ __device__ inline size_t res_smem_bytes(int lx, int ly, int lz, int gtab) {
    const size_t H = (size_t)(lx + 2) * (ly + 2) * (lz + 2);
    const size_t n = (size_t)lx * ly * lz;
    const size_t F = 2 * ((size_t)ly * lz + (size_t)lx * lz + (size_t)lx * ly);
    return 8 * (size_t)gtab + 16 * H + 8 * n + 4 * n + 8 * F + H + 16;
}

// own-node descriptor bits: [0,14) smem index, [14,20) free-neighbour mask
// (x-, x+, y-, y+, z-, z+), [20,25) class, bit 25 brick-surface node.
__device__ __forceinline__ int od_s(int d) { return d & 0x3fff; }
__device__ __forceinline__ int od_mask(int d) { return (d >> 14) & 0x3f; }
__device__ __forceinline__ int od_cls(int d) { return (d >> 20) & 0x1f; }
__device__ __forceinline__ bool od_surf(int d) { return (d >> 25) & 1; }

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// (A_c v)_s for a free own node from the halo'd smem array V.
__device__ __forceinline__ double stencil_smem(const ClassTable& T, const double* V, int s, int cls,
                                               int mk, int SY, int SZ) {
    const double tx_ = ((mk & 1) ? V[s - 1] : 0.0) + ((mk & 2) ? V[s + 1] : 0.0);
    const double ty_ = ((mk & 4) ? V[s - SY] : 0.0) + ((mk & 8) ? V[s + SY] : 0.0);
    const double tz_ = ((mk & 16) ? V[s - SZ] : 0.0) + ((mk & 32) ? V[s + SZ] : 0.0);
    return T.diag[cls] * V[s] - ((T.c[0][cls] * tx_ + T.c[1][cls] * ty_) + T.c[2][cls] * tz_);
}

// scipy's cg operation for operation: two grid barriers per iteration (p.q; then r.z, r.r).
template <bool GAUSS, int NPT>
__global__ void __launch_bounds__(kResTPB, 1) k_pcg_resident(ResParams RP) {
    cg::grid_group grid = cg::this_grid();
    const PcgParams& P = RP.P;
    const Grid& g = P.g;
    __shared__ ClassTable T;
    __shared__ double red[8 * 32];
    __shared__ double tot[8];
    extern __shared__ __align__(16) unsigned char smem[];
    const bool prof = RP.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    int np = 0;
    if (prof) RP.prof[np++] = global_ns();

    // ---- brick of this CTA ----
    const int G = gridDim.x;
    const int b = blockIdx.x;
    const int bxi = b % RP.ng[0], byi = (b / RP.ng[0]) % RP.ng[1], bzi = b / (RP.ng[0] * RP.ng[1]);
    const int x0 = RP.off[0][bxi], y0 = RP.off[1][byi], z0 = RP.off[2][bzi];
    const int lx = RP.off[0][bxi + 1] - x0, ly = RP.off[1][byi + 1] - y0, lz = RP.off[2][bzi + 1] - z0;
    const int LX = lx + 2, LY = ly + 2, LZ = lz + 2;
    const int H = LX * LY * LZ;
    const int SY = LX, SZ = LX * LY;
    const int nown = lx * ly * lz;
    const int fx = ly * lz, fy = lx * lz, fz = lx * ly;
    const int nface = 2 * (fx + fy + fz);

    const int gtab_n = GAUSS ? gauss_smem_len(g) : 0;
    double* tx = reinterpret_cast<double*>(smem);
    double* ty = tx + 6 * g.nc[0];
    double* tz = ty + 6 * g.nc[1];
    double* bx_ = tz + 6 * g.nc[2];
    double* by_ = bx_ + g.NX;
    double* bz_ = by_ + g.NY;
    double* PS = tx + gtab_n;
    double* RS = PS + H;
    double* XS = RS + H;
    int* GID = reinterpret_cast<int*>(XS + nown);
    int* FS = GID + nown;
    int* FG = FS + nface;
    uint8_t* CL = reinterpret_cast<uint8_t*>(FG + nface);

    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    if (GAUSS) build_gauss_tables(g, P.src, tx, ty, tz);
    for (int s = threadIdx.x; s < H; s += kResTPB) {
        const int u = s % LX, v = (s / LX) % LY, w = s / SZ;
        const int i = x0 + u - 1, j = y0 + v - 1, k = z0 + w - 1;
        const bool in = i >= 0 && i <= g.nc[0] && j >= 0 && j <= g.nc[1] && k >= 0 && k <= g.nc[2];
        CL[s] = in ? (uint8_t)class_of(g, i, j, k) : kNoNode;
        PS[s] = 0.0;
        RS[s] = 0.0;
    }
    __syncthreads();
    if (GAUSS) build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
    if (prof) RP.prof[120] = global_ns();
    // halo face cells (the 7-point stencil needs no edge or corner cells)
    for (int e0 = threadIdx.x; e0 < nface; e0 += kResTPB) {
        int e = e0, u, v, w;
        if (e < 2 * fx) {
            const int side = e / fx, r = e % fx;
            u = side ? LX - 1 : 0; v = r % ly + 1; w = r / ly + 1;
        } else if ((e -= 2 * fx) < 2 * fy) {
            const int side = e / fy, r = e % fy;
            v = side ? LY - 1 : 0; u = r % lx + 1; w = r / lx + 1;
        } else {
            e -= 2 * fy;
            const int side = e / fz, r = e % fz;
            w = side ? LZ - 1 : 0; u = r % lx + 1; v = r / lx + 1;
        }
        const int s = u + SY * v + SZ * w;
        const bool in = CL[s] != kNoNode;
        FS[e0] = in ? s : -1;
        FG[e0] = in ? (x0 + u - 1) + g.NX * ((y0 + v - 1) + g.NY * (z0 + w - 1)) : 0;
    }

    // ---- own nodes: descriptors in registers, global ids in smem ----
    int od[NPT];
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        const int nl = threadIdx.x + m * kResTPB;
        od[m] = -1;
        if (nl < nown) {
            const int u = nl % lx + 1, v = (nl / lx) % ly + 1, w = nl / (lx * ly) + 1;
            const int s = u + SY * v + SZ * w;
            const int cls = CL[s];
            int mask = 0;
            const int nb[6] = {s - 1, s + 1, s - SY, s + SY, s - SZ, s + SZ};
#pragma unroll
            for (int e = 0; e < 6; ++e) {
                const int c = CL[nb[e]];
                if (c != kNoNode && T.nd[c] != 0.0) mask |= 1 << e;
            }
            const bool surf = u == 1 || u == lx || v == 1 || v == ly || w == 1 || w == lz;
            od[m] = s | (mask << 14) | (cls << 20) | ((int)surf << 25);
            GID[nl] = (x0 + u - 1) + g.NX * ((y0 + v - 1) + g.NY * (z0 + w - 1));
            XS[nl] = 0.0;
        }
    }

    // ---- phase 0: constrained RHS, r = b, x = 0 ----
    if (GAUSS) __syncthreads();          // Gaussian bounds visible
    if (prof) RP.prof[121] = global_ns();
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        const int p = GID[threadIdx.x + m * kResTPB];
        const int cls = od_cls(od[m]);
        double bv;
        if (T.nd[cls] == 0.0) {
            bv = dirichlet_value(P, p);
        } else {
            int i, j, k;
            decode(g, p, i, j, k);
            bv = T.mass[cls] * P.T[p];
            if (P.load) bv += P.load[p];
            if (GAUSS) bv = add_gaussian(bv, g, tx, ty, tz, bx_, by_, bz_, i, j, k);
            const int sy = g.NX, sz = g.NX * g.NY;
            double lift = 0.0;
            if (i > 0 && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i - 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dirichlet_value(P, p - 1);
            if (i < g.nc[0] && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dirichlet_value(P, p + 1);
            if (j > 0 && T.nd[cls + 3 * (axis_class(j - 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dirichlet_value(P, p - sy);
            if (j < g.nc[1] && T.nd[cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dirichlet_value(P, p + sy);
            if (k > 0 && T.nd[cls + 9 * (axis_class(k - 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dirichlet_value(P, p - sz);
            if (k < g.nc[2] && T.nd[cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dirichlet_value(P, p + sz);
            bv += lift;
        }
        P.b[p] = bv;
        RS[od_s(od[m])] = bv;
        if (od_surf(od[m])) RP.xg[p] = bv;
        const double z = __dmul_rn(T.invd[cls], bv);
        acc[0] += bv * bv;
        acc[1] += bv * z;
    }
    if (prof) RP.prof[122] = global_ns();
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) { P.part[0 * G + b] = acc[0]; P.part[1 * G + b] = acc[1]; }
    grid.sync();
    {
        const int s2[2] = {0, 1};
        grid_sum_fast<2>(P.part, s2, G, tot);
    }
    if (prof) RP.prof[np++] = global_ns();
    const double bb = tot[0];
    double rz = tot[1];
    const double bnorm = sqrt(bb);
    const double atol = P.rtol * bnorm;
    double rnorm = bnorm;
    int it = 0, status = 0;
    double rho_prev = 1.0;

    double q[NPT];
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
            // ---- phase A: halo r in, p = z (+ beta p) on own + halo, q = A_c p ----
#define TL_STX(slot) \
    if (prof && it == 3) RP.prof[slot] = global_ns();
            TL_STX(140)
            double fv[kResKF];
#pragma unroll
            for (int t = 0; t < kResKF; ++t) {      // issue every halo load first
                const int e = threadIdx.x + t * kResTPB;
                fv[t] = (e < nface && FS[e] >= 0) ? __ldcg(RP.xg + FG[e]) : 0.0;
            }
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                if (od[m] < 0) continue;
                const int s = od_s(od[m]);
                const double z = __dmul_rn(T.invd[od_cls(od[m])], RS[s]);
                PS[s] = first ? z : __dadd_rn(__dmul_rn(beta, PS[s]), z);
            }
#pragma unroll
            for (int t = 0; t < kResKF; ++t) {
                const int e = threadIdx.x + t * kResTPB;
                if (e >= nface) break;
                const int s = FS[e];
                if (s < 0) continue;
                RS[s] = fv[t];
                const double z = __dmul_rn(T.invd[CL[s]], fv[t]);
                PS[s] = first ? z : __dadd_rn(__dmul_rn(beta, PS[s]), z);
            }
            TL_STX(141)
            __syncthreads();
            TL_STX(142)
            double pq[1] = {0.0};
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                if (od[m] < 0) continue;
                const int d = od[m], s = od_s(d), cls = od_cls(d);
                const double pp = PS[s];
                const double qv = (T.nd[cls] == 0.0) ? pp : stencil_smem(T, PS, s, cls, od_mask(d), SY, SZ);
                q[m] = qv;
                pq[0] += pp * qv;
            }
            TL_STX(143)
            block_sum<1>(pq, red);
            if (threadIdx.x == 0) P.part[2 * G + b] = pq[0];
            TL_STX(144)
            if (RP.prof && it == 3 && threadIdx.x == 0) RP.prof[256 + b] = global_ns();
            grid.sync();
            TL_STX(145)
            {
                const int s1[1] = {2};
                grid_sum_fast<1>(P.part, s1, G, tot);
            }
            TL_STX(146)
            if (prof && it < 64) RP.prof[np++] = global_ns();
            const double alpha = rho / tot[0];
            // ---- phase B: x += alpha p, r -= alpha q, r.z, r.r; publish surface r ----
            double a2[2] = {0.0, 0.0};
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                if (od[m] < 0) continue;
                const int d = od[m], s = od_s(d), nl = threadIdx.x + m * kResTPB;
                const double xv = __dadd_rn(XS[nl], __dmul_rn(alpha, PS[s]));
                XS[nl] = xv;
                const double rv = __dsub_rn(RS[s], __dmul_rn(alpha, q[m]));
                RS[s] = rv;
                if (od_surf(d)) {
                    // r for the next iteration's halo; x speculatively, for the final residual
                    RP.xg[GID[nl]] = rv;
                    RP.xx[GID[nl]] = xv;
                }
                const double z = __dmul_rn(T.invd[od_cls(d)], rv);
                a2[0] += rv * z;
                a2[1] += rv * rv;
            }
            TL_STX(147)
            block_sum<2>(a2, red);
            if (threadIdx.x == 0) { P.part[0 * G + b] = a2[0]; P.part[1 * G + b] = a2[1]; }
            TL_STX(148)
            grid.sync();
            TL_STX(149)
            {
                const int s2[2] = {0, 1};
                grid_sum_fast<2>(P.part, s2, G, tot);
            }
            TL_STX(150)
#undef TL_STX
            if (prof && it < 64) RP.prof[np++] = global_ns();
            rz = tot[0];
            rnorm = sqrt(tot[1]);
            rho_prev = rho;
            ++it;
        }
    }

    // ---- true residual ||A_c x - b||: surface x was published by the last phase B
    //      (before the barrier that ended the loop); gather the halo x into PS ----
    __syncthreads();
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        PS[od_s(od[m])] = XS[threadIdx.x + m * kResTPB];
    }
#pragma unroll
    for (int t = 0; t < kResKF; ++t) {
        const int e = threadIdx.x + t * kResTPB;
        if (e < nface && FS[e] >= 0) PS[FS[e]] = it > 0 ? __ldcg(RP.xx + FG[e]) : 0.0;
    }
    __syncthreads();
    double res[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        const int d = od[m], s = od_s(d), cls = od_cls(d);
        const int p = GID[threadIdx.x + m * kResTPB];
        const double xp = PS[s];
        const double ax = (T.nd[cls] == 0.0) ? xp : stencil_smem(T, PS, s, cls, od_mask(d), SY, SZ);
        const double bv = P.b[p];
        const double dd = ax - bv;
        res[0] += dd * dd;
        res[1] += isfinite(xp) ? 0.0 : 1.0;
        P.T[p] = (T.nd[cls] == 0.0) ? bv : xp;      // x_D = g = b_D (fem.py:289-290)
    }
    block_sum<2>(res, red);
    if (threadIdx.x == 0) { P.part[0 * G + b] = res[0]; P.part[3 * G + b] = res[1]; }
    grid.sync();
    {
        const int s2[2] = {0, 3};
        grid_sum_fast<2>(P.part, s2, G, tot);
    }
    if (b == 0 && threadIdx.x == 0) {
        const double tres = bnorm > 0.0 ? sqrt(tot[0]) / bnorm : 0.0;
        if (status == 0 && tot[1] > 0.0) status = 3;
        if (status == 0 && (!isfinite(tres) || tres > 1e2 * P.rtol)) status = 2;
        P.info->iterations = (status == 1) ? P.maxiter : it;
        P.info->status = status;
        P.info->bnorm = bnorm;
        P.info->rnorm = rnorm;
        P.info->true_resid = tres;
        if (prof) { RP.prof[np++] = global_ns(); RP.prof[127] = np; }
    }
}

}  // namespace tl
