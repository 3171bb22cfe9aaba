// tl_vc.cuh — temperature-dependent implicit step, sm_100a, fp64.
//
// assemble_system (lpbfsim/fem.py:129-194) with _material_arrays (:214-238), the secant
// latent capacity (:197-211) and the lumped convection / lagged-radiation top terms
// (_add_robin, :241-268), then constrained (:89-105) + Jacobi-PCG with scipy's
// recurrences (solve_linear, :271-291).  The Picard loop (:307-355) drives one call of
// tl_vc_step_host per pass.
//
// On a Kuhn tet the P1 gradients are axis-aligned along the tet's path (000 -> +e_p0 ->
// +e_p1 -> 111), so kbar vol grad_i.grad_j couples only consecutive path vertices and the
// assembled operator is a 7-point stencil with per-edge weights (oracle/varcoef.py):
//     (A x)_p = diag_p x_p - sum_a (w_a[p] x_{p+e_a} + w_a[p-e_a] x_{p-e_a}).
// k_vc_assemble computes diag, w and b node by node (gather over the 24 tets touching the
// node: no atomics, deterministic); k_vc_cg runs the whole Jacobi-PCG in one cooperative
// launch (two grid barriers per iteration) with fixed-order reductions.  This path is a seam-3
// solver (host buffers in and out), not the device-resident two-level loop.
#pragma once

#include "tl_kernels.cuh"

namespace tl {

struct VcMat {
    const double *kT, *kv, *cT, *cv;
    int nk, nc;
    double rho, chi, S, Tm;
    int latent;
};

// PiecewiseMaterial (materials.py:161-190) over a box region (runner.py:141-151: the tets
// whose centroid lies in the closed local box take the inside material), and a latent
// mask restricted to that region (latent_reference local).
struct VcRegion {
    double lo[3], hi[3];
    int piecewise;       // 1: inside tets use Mi, outside Mo
    int latent_inside;   // 1: latent term only on inside tets
};

struct VcRobin {
    double h, se, Tamb;
    int on;
};

__device__ __forceinline__ double vc_interp(double x, const double* xp, const double* fp, int n) {
    return tab_interp(x, xp, fp, n);
}

// tanh saturates to +-1 exactly in fp64 beyond |a| ~ 19.1 (1 - tanh(22) = 1.6e-19 < ulp / 2):
// the shortcut returns the same bits and spares the cold bulk of the plate two tanh calls
// per quadrature point.
__device__ __forceinline__ double vc_phase(const VcMat& M, double T) {
    const double a = M.S * (T - M.Tm);
    if (a > 22.0) return 1.0;
    if (a < -22.0) return 0.0;
    return 0.5 * (1.0 + tanh(a));
}

__device__ __forceinline__ double vc_phase_deriv(const VcMat& M, double T) {
    const double ax = fabs(M.S * (T - M.Tm));
    const double e = exp(-ax);
    const double s = 2.0 * e / (1.0 + e * e);
    return 0.5 * M.S * (s * s);
}

// _latent_slope: chi * secant of the liquid fraction over the step
__device__ __forceinline__ double vc_latent(const VcMat& M, double T, double T_old) {
    const double dT = T - T_old;
    if (fabs(dT) < 1e-6) return M.chi * vc_phase_deriv(M, 0.5 * (T + T_old));
    return M.chi * ((vc_phase(M, T) - vc_phase(M, T_old)) / dT);
}

// Phase 1, one thread per (cell, tet): kbar, the lumped mass of each vertex (times vol)
// and the Gaussian load of each vertex (times vol), stored per tet so every tet's
// quadrature-point material evaluations run once (not once per touching node).
// The (T, value) tables of a material staged in shared memory (the np.interp searches are
// chains of dependent loads: 8 per quadrature point); `at` holds 2 (nk + nc) doubles.
__device__ __forceinline__ VcMat vc_stage_tables(const VcMat& M, double* at) {
    for (int e = threadIdx.x; e < M.nk; e += blockDim.x) { at[e] = M.kT[e]; at[M.nk + e] = M.kv[e]; }
    for (int e = threadIdx.x; e < M.nc; e += blockDim.x) { at[2 * M.nk + e] = M.cT[e]; at[2 * M.nk + M.nc + e] = M.cv[e]; }
    VcMat S = M;
    S.kT = at; S.kv = at + M.nk; S.cT = at + 2 * M.nk; S.cv = at + 2 * M.nk + M.nc;
    return S;
}

__global__ void k_vc_tets(Grid g, VcMat Mi_g, VcMat Mo_g, VcRegion R, const double* __restrict__ T_old,
                          const double* __restrict__ T_lag, double dt, Gauss src, double* __restrict__ tk,
                          double* __restrict__ tml, double* __restrict__ tsrc) {
    extern __shared__ double vc_tab[];           // 2 (nk + nc) of Mi, then of Mo (piecewise only)
    const VcMat Mi = vc_stage_tables(Mi_g, vc_tab);
    const VcMat Mo = R.piecewise ? vc_stage_tables(Mo_g, vc_tab + 2 * (Mi_g.nk + Mi_g.nc)) : Mi;
    __syncthreads();
    const double A = TL_QA, B = TL_QB;
    const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int st[3] = {1, g.NX, g.NX * g.NY};
    const int ncell = g.nc[0] * g.nc[1] * g.nc[2];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 6 * ncell; e += gridDim.x * blockDim.x) {
        const int c = e / 6, t = e - 6 * c;
        const int ci = c % g.nc[0], cr = c / g.nc[0];
        const int cell[3] = {ci, cr % g.nc[1], cr / g.nc[1]};
        const int c0 = cell[0] + g.NX * (cell[1] + g.NY * cell[2]);
        int off[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int v = 1; v < 4; ++v) {
            for (int a = 0; a < 3; ++a) off[v][a] = off[v - 1][a];
            off[v][perms[t][v - 1]] += 1;
        }
        double Tl[4], To[4];
        for (int v = 0; v < 4; ++v) {
            const int id = c0 + off[v][0] * st[0] + off[v][1] * st[1] + off[v][2] * st[2];
            Tl[v] = T_lag[id];
            To[v] = T_old[id];
        }
        bool inside = true;
        if (R.piecewise || R.latent_inside) {
            for (int a = 0; a < 3; ++a) {
                double sx = 0.0;
                for (int v = 0; v < 4; ++v) sx += node_coord(g, a, cell[a] + off[v][a]);
                const double cen = sx / 4.0;
                inside = inside && cen >= R.lo[a] && cen <= R.hi[a];
            }
        }
        const VcMat& M = (R.piecewise && !inside) ? Mo : Mi;
        const bool lat_on = M.latent && (!R.latent_inside || inside);
        double kbar = 0.0, ml[4] = {0.0, 0.0, 0.0, 0.0}, qs[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < 4; ++q) {
            double tq = 0.0, tqo = 0.0;
            for (int v = 0; v < 4; ++v) {
                const double ph = (v == q) ? A : B;
                tq += ph * Tl[v];
                tqo += ph * To[v];
            }
            const double kq = vc_interp(tq, M.kT, M.kv, M.nk);
            double cq = vc_interp(tq, M.cT, M.cv, M.nc);
            if (lat_on) cq += vc_latent(M, tq, tqo);
            kbar += 0.25 * kq;
            const double mq = 0.25 * (M.rho * cq / dt);
            double Qq = 0.0;
            if (src.on) {
                double x[3];
                for (int a = 0; a < 3; ++a) {
                    double sx = 0.0;
                    for (int v = 0; v < 4; ++v) sx += ((v == q) ? A : B) * node_coord(g, a, cell[a] + off[v][a]);
                    x[a] = sx;
                }
                const double ex = 3.0 * ((x[0] - src.center[0]) / src.radius) * ((x[0] - src.center[0]) / src.radius);
                const double ey = 3.0 * ((x[1] - src.center[1]) / src.radius) * ((x[1] - src.center[1]) / src.radius);
                const double ez = 3.0 * ((x[2] - src.center[2]) / src.depth) * ((x[2] - src.center[2]) / src.depth);
                // exp(-a) is exactly 0 for a > 745.14: the same bits without the call far from the beam
                const double ea = ex + ey + ez;
                Qq = ea > 745.2 ? 0.0 : 0.25 * (src.peak * exp(-ea));
            }
            for (int r = 0; r < 4; ++r) {
                const double phr = (r == q) ? A : B;
                ml[r] += mq * phr;
                qs[r] += Qq * phr;
            }
        }
        tk[e] = kbar;
        for (int r = 0; r < 4; ++r) {
            tml[4 * (size_t)e + r] = ml[r] * vol;
            tsrc[4 * (size_t)e + r] = qs[r] * vol;
        }
    }
}

// Phase 2, one thread per node: gather the 24 touching tets (fixed order, no atomics).
__global__ void k_vc_assemble(Grid g, const double* __restrict__ tk, const double* __restrict__ tml,
                              const double* __restrict__ tsrc, const double* __restrict__ T_old,
                              const double* __restrict__ T_lag, const double* __restrict__ extra, VcRobin rb,
                              double* __restrict__ diag, double* __restrict__ wx, double* __restrict__ wy,
                              double* __restrict__ wz, double* __restrict__ b) {
    const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
        int idx[3];
        decode(g, p, idx[0], idx[1], idx[2]);
        const double Top = T_old[p];
        double dg = 0.0, bb = 0.0, wf[3] = {0.0, 0.0, 0.0};
        for (int o = 0; o < 8; ++o) {
            const int oo[3] = {o & 1, (o >> 1) & 1, (o >> 2) & 1};
            int cell[3];
            bool ok = true;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                cell[a] = idx[a] - oo[a];
                ok = ok && cell[a] >= 0 && cell[a] < g.nc[a];
            }
            if (!ok) continue;
            const int c = cell[0] + g.nc[0] * (cell[1] + g.nc[1] * cell[2]);
            for (int t = 0; t < 6; ++t) {
                int off[3] = {0, 0, 0}, r = -1;
                for (int v = 0; v < 4; ++v) {
                    if (v > 0) off[perms[t][v - 1]] += 1;
                    if (off[0] == oo[0] && off[1] == oo[1] && off[2] == oo[2]) r = v;
                }
                if (r < 0) continue;
                const size_t e = 6 * (size_t)c + t;
                const double ml = tml[4 * e + r];
                const double kbar = tk[e];
                dg += ml;
                bb += ml * Top + tsrc[4 * e + r];
                if (r > 0) {
                    const int ax = perms[t][r - 1];
                    dg += kbar * vol / (g.h[ax] * g.h[ax]);
                }
                if (r < 3) {
                    const int ax = perms[t][r];
                    const double we = kbar * vol / (g.h[ax] * g.h[ax]);
                    dg += we;
                    wf[ax] += we;
                }
            }
        }
        if (rb.on && idx[2] == g.nc[2]) {
            // top triangles (0,0)-(1,0)-(1,1) and (0,0)-(0,1)-(1,1) of the top-layer cells
            const int tri[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {0, 1}, {1, 1}}};
            const double area = 0.5 * g.h[0] * g.h[1];
            const double load = rb.h * rb.Tamb + rb.se * (rb.Tamb * rb.Tamb * rb.Tamb * rb.Tamb);
            for (int cj = idx[1] - 1; cj <= idx[1]; ++cj) {
                for (int ci = idx[0] - 1; ci <= idx[0]; ++ci) {
                    if (ci < 0 || cj < 0 || ci >= g.nc[0] || cj >= g.nc[1]) continue;
                    for (int t = 0; t < 2; ++t) {
                        int me = -1, vid[3];
                        for (int v = 0; v < 3; ++v) {
                            const int vi = ci + tri[t][v][0], vj = cj + tri[t][v][1];
                            vid[v] = vi + g.NX * (vj + g.NY * idx[2]);
                            if (vi == idx[0] && vj == idx[1]) me = v;
                        }
                        if (me < 0) continue;
                        for (int v = 0; v < 3; ++v) {
                            if (v == me) continue;
                            const double tq = 0.5 * (T_lag[vid[me]] + T_lag[vid[v]]);
                            const double coeff = rb.h + rb.se * (tq * tq * tq);
                            dg += coeff * 0.5 * area / 3.0;
                            bb += load * 0.5 * area / 3.0;
                        }
                    }
                }
            }
        }
        if (extra) bb += extra[p];
        diag[p] = dg;
        wx[p] = wf[0];
        wy[p] = wf[1];
        wz[p] = wf[2];
        b[p] = bb;
    }
}

// constrained(): free rows take their Dirichlet couplings into b; Dirichlet rows -> identity
__global__ void k_vc_constrain_b(Grid g, const unsigned char* __restrict__ dm, const double* __restrict__ gv,
                                 const double* __restrict__ wx, const double* __restrict__ wy,
                                 const double* __restrict__ wz, double* __restrict__ diag, double* __restrict__ b) {
    const int st[3] = {1, g.NX, g.NX * g.NY};
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
        if (dm[p]) { b[p] = gv[p]; diag[p] = 1.0; continue; }
        int idx[3];
        decode(g, p, idx[0], idx[1], idx[2]);
        const double* w[3] = {wx, wy, wz};
        double add = 0.0;
        for (int a = 0; a < 3; ++a) {
            if (idx[a] < g.nc[a] && dm[p + st[a]]) add += w[a][p] * gv[p + st[a]];
            if (idx[a] > 0 && dm[p - st[a]]) add += w[a][p - st[a]] * gv[p - st[a]];
        }
        b[p] += add;
    }
}

__global__ void k_vc_constrain_w(Grid g, const unsigned char* __restrict__ dm, double* __restrict__ wx,
                                 double* __restrict__ wy, double* __restrict__ wz) {
    const int st[3] = {1, g.NX, g.NX * g.NY};
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
        int idx[3];
        decode(g, p, idx[0], idx[1], idx[2]);
        double* w[3] = {wx, wy, wz};
        for (int a = 0; a < 3; ++a)
            if (dm[p] || (idx[a] < g.nc[a] && dm[p + st[a]])) w[a][p] = 0.0;
    }
}

__device__ __forceinline__ double vc_apply(const Grid& g, const double* diag, const double* wx, const double* wy,
                                           const double* wz, const double* x, int p) {
    int i, j, k;
    decode(g, p, i, j, k);
    const int sy = g.NX, sz = g.NX * g.NY;
    double y = diag[p] * x[p];
    if (i < g.nc[0]) y -= wx[p] * x[p + 1];
    if (i > 0) y -= wx[p - 1] * x[p - 1];
    if (j < g.nc[1]) y -= wy[p] * x[p + sy];
    if (j > 0) y -= wy[p - sy] * x[p - sy];
    if (k < g.nc[2]) y -= wz[p] * x[p + sz];
    if (k > 0) y -= wz[p - sz] * x[p - sz];
    return y;
}

// Jacobi-PCG with scipy's recurrences (solve_linear cg, fem.py:271-298) in ONE cooperative
// launch with TWO grid barriers per iteration:
//   U: x += alpha p, r -= alpha q (the previous iteration's update), z = invd r, partials
//      of r.r and r.z                                          -> barrier, sums
//   P: p = z (first) or p beta + z (scipy's two roundings), written to the other buffer
//      of a ping-pong pair; q = A p with the neighbours' new p recomputed from their z and
//      old p (bitwise the owners' values), partial of p.q     -> barrier, sum
// Every reduction is a fixed-order block tree plus a fixed-order sum of the block
// partials that every CTA performs identically (grid_sum), so all CTAs take the same
// branch and the result is deterministic.  part: 6 slots of gridDim.x.
struct VcCg {
    const double *diag, *wx, *wy, *wz, *b;
    const unsigned char* dm;
    const double* g;
    double *x, *r, *z, *p, *q, *part;     // p: 2 n (ping-pong)
    double rtol;
    int maxiter;
    SolveInfoDev* info;
};

__device__ __forceinline__ double vc_pnew(const double* z, const double* pold, double beta, bool first, int j) {
    return first ? z[j] : __dadd_rn(__dmul_rn(pold[j], beta), z[j]);
}

__global__ void __launch_bounds__(256) k_vc_cg(Grid G, VcCg C) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[64];
    __shared__ double tot[2];
    const int n = G.n, NB = gridDim.x, b = blockIdx.x;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x, ts = gridDim.x * blockDim.x;
    const int sy = G.NX, sz = G.NX * G.NY;
    // ||b||, x = 0, r = b
    {
        double v[1] = {0.0};
        for (int i = t0; i < n; i += ts) {
            const double bv = C.b[i];
            C.x[i] = 0.0;
            C.r[i] = bv;
            v[0] += bv * bv;
        }
        block_sum<1>(v, red);
        if (threadIdx.x == 0) C.part[0 * NB + b] = v[0];
    }
    grid.sync();
    { const int s1[1] = {0}; grid_sum<1>(C.part, s1, NB, tot); }
    const double bnorm = sqrt(tot[0]);
    double rr = tot[0], rho_prev = 1.0, alpha = 0.0;
    int it = 0, status = 0;
    if (bnorm > 0.0) {
        const double atol = C.rtol * bnorm;
        status = 1;
        for (; it <= C.maxiter; ++it) {
            double* pcur = C.p + (size_t)(it & 1) * n;          // p of iteration it-1 (read)
            double* pnew = C.p + (size_t)((it + 1) & 1) * n;    // p of iteration it (written)
            // U
            double v[2] = {0.0, 0.0};
            for (int i = t0; i < n; i += ts) {
                double rv = C.r[i];
                if (it > 0) {
                    C.x[i] += alpha * pcur[i];
                    rv = rv - alpha * C.q[i];
                    C.r[i] = rv;
                }
                const double zz = (1.0 / C.diag[i]) * rv;
                C.z[i] = zz;
                v[0] += rv * rv;
                v[1] += rv * zz;
            }
            block_sum<2>(v, red);
            if (threadIdx.x == 0) { C.part[1 * NB + b] = v[0]; C.part[2 * NB + b] = v[1]; }
            grid.sync();
            { const int s2[2] = {1, 2}; grid_sum<2>(C.part, s2, NB, tot); }
            if (it > 0) rr = tot[0];
            if (it == C.maxiter) { status = 1; break; }      // scipy: no test after the last update
            if (!isfinite(rr)) { status = 3; break; }
            if (sqrt(rr) < atol) { status = 0; break; }
            const double rho = tot[1];
            const bool first = it == 0;
            const double beta = first ? 0.0 : rho / rho_prev;
            // P
            double w1[1] = {0.0};
            for (int i = t0; i < n; i += ts) {
                int ii, jj, kk;
                decode(G, i, ii, jj, kk);
                const double pi = vc_pnew(C.z, pcur, beta, first, i);
                pnew[i] = pi;
                double y = C.diag[i] * pi;
                if (ii < G.nc[0]) y -= C.wx[i] * vc_pnew(C.z, pcur, beta, first, i + 1);
                if (ii > 0) y -= C.wx[i - 1] * vc_pnew(C.z, pcur, beta, first, i - 1);
                if (jj < G.nc[1]) y -= C.wy[i] * vc_pnew(C.z, pcur, beta, first, i + sy);
                if (jj > 0) y -= C.wy[i - sy] * vc_pnew(C.z, pcur, beta, first, i - sy);
                if (kk < G.nc[2]) y -= C.wz[i] * vc_pnew(C.z, pcur, beta, first, i + sz);
                if (kk > 0) y -= C.wz[i - sz] * vc_pnew(C.z, pcur, beta, first, i - sz);
                C.q[i] = y;
                w1[0] += pi * y;
            }
            block_sum<1>(w1, red);
            if (threadIdx.x == 0) C.part[3 * NB + b] = w1[0];
            grid.sync();
            { const int s1[1] = {3}; grid_sum<1>(C.part, s1, NB, tot); }
            alpha = rho / tot[0];
            rho_prev = rho;
        }
    }
    // true residual ||A x - b|| / ||b||, then x_D = g
    double v[1] = {0.0};
    for (int i = t0; i < n; i += ts) {
        const double d = vc_apply(G, C.diag, C.wx, C.wy, C.wz, C.x, i) - C.b[i];
        v[0] += d * d;
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0) C.part[4 * NB + b] = v[0];
    grid.sync();
    { const int s1[1] = {4}; grid_sum<1>(C.part, s1, NB, tot); }
    for (int i = t0; i < n; i += ts)
        if (C.dm[i]) C.x[i] = C.g[i];
    if (b == 0 && threadIdx.x == 0) {
        const double tres = bnorm > 0.0 ? sqrt(tot[0]) / bnorm : 0.0;
        if (status == 0 && bnorm > 0.0 && (!isfinite(tres) || tres > 1e2 * C.rtol)) status = 2;
        C.info->iterations = it;
        C.info->status = status;
        C.info->bnorm = bnorm;
        C.info->rnorm = sqrt(rr);
        C.info->true_resid = tres;
    }
}

// Picard control on the device (fem.py:346-354): partials of ||x - T_lag||^2 and ||x||^2,
// and the damped lag update T_lag += theta (x - T_lag).
__global__ void k_vc_inc(int n, const double* __restrict__ x, const double* __restrict__ Tl, double* part) {
    __shared__ double red[64];
    double v[2] = {0.0, 0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double d = x[i] - Tl[i];
        v[0] += d * d;
        v[1] += x[i] * x[i];
    }
    block_sum<2>(v, red);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = v[0]; part[2 * blockIdx.x + 1] = v[1]; }
}

__global__ void k_vc_lag(int n, double theta, const double* __restrict__ x, double* __restrict__ Tl) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Tl[i] = Tl[i] + theta * (x[i] - Tl[i]);
}

// ---------------------------------------------------------------------------------
// Full-mode overlap feedback (twolevel.py:186-239), gathered per global node: over the 24
// global tets touching the node and their 4 quadrature points x_q (mesh.py:116-128) that
// lie in the local box (Box.contains, closed), the local field is located (Kuhn-P1,
// p1_locate on the local lattice) and
//   density = -(c_eff_l rho_l k_g/k_l - c_g rho_g) dT/dt
//             + ((k_g/k_l) dk_l/dT - dk_g/dT) |grad T|^2  [+ (k_g/k_l - 1) Q(x_q)]
// with c_eff = c + chi f'(T) (materials.effective_capacity) and dk/dT the table segment
// slope (zero outside the table), scattered as w_q vol density phi_i(x_q).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double vc_dkdT(double T, const double* xp, const double* fp, int n) {
    if (T <= xp[0] || T >= xp[n - 1]) return 0.0;
    int lo = 0, hi = n - 1;                 // searchsorted(right) - 1
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xp[mid] <= T) lo = mid; else hi = mid;
    }
    return (fp[lo + 1] - fp[lo]) / (xp[lo + 1] - xp[lo]);
}

__global__ void k_overlap_feedback(Grid G, Grid L, const double* __restrict__ Tn, const double* __restrict__ To,
                                   double dt, VcMat Mg, VcMat Ml, Gauss src, double* __restrict__ load) {
    const double A = TL_QA, B = TL_QB;
    const double vol = G.h[0] * G.h[1] * G.h[2] / 6.0;
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    double llo[3], lhi[3];
    for (int a = 0; a < 3; ++a) {
        llo[a] = node_coord(L, a, 0);
        lhi[a] = node_coord(L, a, L.nc[a]);
    }
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < G.n; p += gridDim.x * blockDim.x) {
        int idx[3];
        decode(G, p, idx[0], idx[1], idx[2]);
        double acc = 0.0;
        for (int o = 0; o < 8; ++o) {
            const int oo[3] = {o & 1, (o >> 1) & 1, (o >> 2) & 1};
            int cell[3];
            bool ok = true;
            for (int a = 0; a < 3; ++a) {
                cell[a] = idx[a] - oo[a];
                ok = ok && cell[a] >= 0 && cell[a] < G.nc[a];
            }
            if (!ok) continue;
            for (int t = 0; t < 6; ++t) {
                int off[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                int r = -1;
                for (int v = 0; v < 4; ++v) {
                    if (v > 0) {
                        for (int a = 0; a < 3; ++a) off[v][a] = off[v - 1][a];
                        off[v][perms[t][v - 1]] += 1;
                    }
                    if (off[v][0] == oo[0] && off[v][1] == oo[1] && off[v][2] == oo[2]) r = v;
                }
                if (r < 0) continue;
                for (int q = 0; q < 4; ++q) {
                    double x[3];
                    bool in = true;
                    for (int a = 0; a < 3; ++a) {
                        double sx = 0.0;
                        for (int v = 0; v < 4; ++v) sx += ((v == q) ? A : B) * node_coord(G, a, cell[a] + off[v][a]);
                        x[a] = sx;
                        in = in && x[a] >= llo[a] && x[a] <= lhi[a];
                    }
                    if (!in) continue;
                    // locate in the local lattice: cell, descending fractional order, barycentrics
                    int c[3];
                    double xi[3];
                    for (int a = 0; a < 3; ++a) {
                        int ci = (int)floor((x[a] - (L.lo0[a] + L.off[a])) / L.h[a]);
                        ci = ci < 0 ? 0 : (ci > L.nc[a] - 1 ? L.nc[a] - 1 : ci);
                        c[a] = ci;
                        xi[a] = (x[a] - node_coord(L, a, ci)) / L.h[a];
                    }
                    int o0 = 0, o1 = 1, o2 = 2;
                    if (xi[o1] > xi[o0]) { int tt = o0; o0 = o1; o1 = tt; }
                    if (xi[o2] > xi[o1]) { int tt = o1; o1 = o2; o2 = tt; }
                    if (xi[o1] > xi[o0]) { int tt = o0; o0 = o1; o1 = tt; }
                    const int st[3] = {1, L.NX, L.NX * L.NY};
                    const int n0 = c[0] + L.NX * (c[1] + L.NY * c[2]);
                    const int n1 = n0 + st[o0], n2 = n1 + st[o1], n3 = n2 + st[o2];
                    const double w0 = 1.0 - xi[o0], w1 = xi[o0] - xi[o1], w2 = xi[o1] - xi[o2], w3 = xi[o2];
                    const double Tq = w0 * Tn[n0] + w1 * Tn[n1] + w2 * Tn[n2] + w3 * Tn[n3];
                    const double Tqo = w0 * To[n0] + w1 * To[n1] + w2 * To[n2] + w3 * To[n3];
                    double gr[3];
                    gr[o0] = (Tn[n1] - Tn[n0]) / L.h[o0];
                    gr[o1] = (Tn[n2] - Tn[n1]) / L.h[o1];
                    gr[o2] = (Tn[n3] - Tn[n2]) / L.h[o2];
                    const double gsq = gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2];
                    const double kg = tab_interp(Tq, Mg.kT, Mg.kv, Mg.nk);
                    const double kl = tab_interp(Tq, Ml.kT, Ml.kv, Ml.nk);
                    const double ratio = kg / kl;
                    const double ceff = tab_interp(Tq, Ml.cT, Ml.cv, Ml.nc) + Ml.chi * vc_phase_deriv(Ml, Tq);
                    const double cg = tab_interp(Tq, Mg.cT, Mg.cv, Mg.nc);
                    const double cap = ceff * Ml.rho * ratio - cg * Mg.rho;
                    double dens = -cap * ((Tq - Tqo) / dt);
                    dens += (ratio * vc_dkdT(Tq, Ml.kT, Ml.kv, Ml.nk) - vc_dkdT(Tq, Mg.kT, Mg.kv, Mg.nk)) * gsq;
                    if (src.on) {
                        const double ex = 3.0 * ((x[0] - src.center[0]) / src.radius) * ((x[0] - src.center[0]) / src.radius);
                        const double ey = 3.0 * ((x[1] - src.center[1]) / src.radius) * ((x[1] - src.center[1]) / src.radius);
                        const double ez = 3.0 * ((x[2] - src.center[2]) / src.depth) * ((x[2] - src.center[2]) / src.depth);
                        dens += (ratio - 1.0) * (src.peak * exp(-(ex + ey + ez)));
                    }
                    acc += 0.25 * vol * dens * ((r == q) ? A : B);
                }
            }
        }
        load[p] = acc;
    }
}

}  // namespace tl
