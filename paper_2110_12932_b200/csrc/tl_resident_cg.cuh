// tl_resident_cg.cuh — one-barrier-per-iteration resident PCG (Chronopoulos-Gear), sm_100a fp64.
//
// One launch runs a list of solves back to back (SolveSpec): the micro steps and the
// corrector of a macro step share the CTA setup (node classes, halo lists) and keep the
// evolving local field x in shared memory from one solve to the next.
//
// Same operator, RHS, preconditioner, stopping rule (||r|| < rtol ||b|| tested at the top
// of each iteration on the directly computed r.r) and final checks as scipy's cg /
// k_pcg_resident, but the Chronopoulos-Gear recurrences
//     u = M r, w = A u, gamma = r.u, delta = w.u
//     beta = gamma/gamma_prev, alpha = gamma/(delta - beta gamma/alpha_prev)
//     p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s
// put the three dots of an iteration in ONE reduction, so each iteration needs one grid
// barrier instead of two.  In exact arithmetic the iterates equal CG's; in fp64 they
// agree with scipy's to ~4e-16 with identical iteration counts on the golden systems
// (tests/test_oracle_golden.py::test_chronopoulos_gear_matches_scipy_cg).
//
// Data placement per CTA brick: u with a one-node halo (the stencil input), r and s of
// own nodes and of the halo face cells (advanced by the same recurrences as their
// owners), w of own nodes in registers, x and p of own nodes in shared memory.
// Only the brick-surface w values cross CTAs (ping-pong exchange buffers).
//
// Shared memory: [US: H][RO: n][SO: n][XO: n, unless xglob][PO: n (+ Gaussian tables overlay during phase 0)]
//                [RF: F][SF: F][GID: n int][FS: F int][FG: F int][CL: H bytes]
#pragma once

#include "tl_resident.cuh"

namespace tl {

// One solve of a multi-solve launch (all micro steps + corrector of a macro step).
struct SolveSpec {
    double mbase;                 // (rho c / dt) V / 24 of this step
    double w;                     // trace blend weight of the Dirichlet data (1-w) gA + w gB
    Gauss src;                    // Gaussian at this step's t1 (src.on == 0: none)
    int tin;                      // T_old: 0 = P.T (global), 1 = previous solve's x, 2 = saved copy
    int save_before;              // 1: save T_old of this solve (before_final, multirate.py:136-137)
    int tout;                     // 1: write the result to P.T
    SolveInfoDev* info;           // this solve's outcome record
    double* snap;                 // optional copy of the result (recorder snapshots), or nullptr
    const double* load;           // this solve's precomputed Gaussian load over box (or nullptr)
    int box[6];                   // [i0, i1) x [j0, j1) x [k0, k1): nodes whose Gaussian term can
                                  // change the RHS; load is dense over it (x fastest)
};

struct ResCGParams {
    PcgParams P;                  // grid, cbase, gA/gB, g_const, load, b, part, rtol, maxiter
    double* xr;                   // exchange: brick-surface r0 / final x, n doubles
    double* xw;                   // exchange: brick-surface w, 2 n doubles (ping-pong)
    double* saved;                // n doubles: T_old saved for the corrector
    const SolveSpec* specs;       // nspec solves run back to back in one launch, or nullptr:
    int nspec;                    // one solve described by spec0 (kernel parameter, no copy)
    SolveSpec spec0;
    unsigned long long* prof;
    int ng[3];
    int off[3][kResMaxSplit + 1];
    // static per-CTA setup (node classes, halo face lists, node descriptors) cached in
    // global memory across solves of one grid: sc_mode 0 = compute, 1 = compute and store,
    // 2 = load (the setup depends only on the grid shape and the brick plan)
    int* scache;
    long long sc_stride;
    int sc_mode;
    // !MULTI: the residual partials are reduced by the last CTA to finish (no second grid
    // barrier at the end of the solve); counter zero between launches
    unsigned* tail_count;
    // launch-persistent arrival counter of grid_allreduce (nullptr: cg grid.sync)
    unsigned* bar_count;
    // own-node x in global memory (CTA b at xglob + b * xg_stride), or nullptr: in SMEM
    double* xglob;
    long long xg_stride;
};

// xglob: x of the own nodes kept in global memory (L2) instead of SMEM, for bricks that
// would not fit otherwise (the cfg2 global grid); x is touched once per iteration.
__host__ __device__ inline size_t rescg_smem_bytes(int lx, int ly, int lz, int gtab, bool xglob = false) {
    const size_t H = (size_t)(lx + 2) * (ly + 2) * (lz + 2);
    const size_t n = (size_t)lx * ly * lz;
    const size_t F = 2 * ((size_t)ly * lz + (size_t)lx * lz + (size_t)lx * ly);
    const size_t extra = (size_t)gtab > n ? (size_t)gtab - n : 0;   // tables overlay PO
    return 8 * extra + 9 * H + (xglob ? 28 : 36) * n + 24 * F + 16;
}

// Block reduction + grid barrier + grid reduction in one pass (replaces block_sum,
// grid.sync and grid_sum_fast, saving their extra __syncthreads): warp 0 of each CTA
// publishes the CTA partials, arrives with a release increment of a launch-persistent
// counter, polls it with acquire loads until all G CTAs of this epoch arrived, then sums
// the G partials in the same fixed order in every CTA (deterministic, bitwise equal).
template <int NV>
__device__ __forceinline__ void grid_allreduce(double (&v)[NV], double* red, double* part, int G,
                                               unsigned* cnt, unsigned target, double* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
        double sv[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) sv[k] = warp_sum(lane < nw ? red[k * 32 + lane] : 0.0);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < NV; ++k) part[k * G + blockIdx.x] = sv[k];
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        }
        unsigned c;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(cnt) : "memory");
        } while ((int)(c - target) < 0);
        constexpr int PL = 5;                  // G <= 160
        double pv[NV][PL];
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int t = 0; t < PL; ++t) {
                const int bb = lane + 32 * t;
                pv[k][t] = bb < G ? __ldcg(part + k * G + bb) : 0.0;
            }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < PL; ++t) acc += pv[k][t];
            acc = warp_sum(acc);
            if (lane == 0) tot[k] = acc;
        }
    }
    __syncthreads();
}

// MULTI = false: exactly one solve (specs[0]); the solve loop folds away, which keeps the
// kernel at ~106 registers without spills.
template <bool GAUSS, int NPT, bool MULTI, bool XG = false>
__global__ void __launch_bounds__(kResTPB, 1) k_pcg_resident_cg(ResCGParams RP) {
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
    if (RP.prof && threadIdx.x == 0 && blockIdx.x < 256) RP.prof[768 + blockIdx.x] = global_ns();   // CTA start

    const int G = gridDim.x;
    const int b = blockIdx.x;
    // grid_allreduce epochs count from the counter value before this launch's first
    // grid.sync (no CTA can arrive at a grid_allreduce before every CTA passed that sync)
    unsigned bar_target = RP.bar_count ? __ldcg(RP.bar_count) : 0u;
    // the CG loop has ONE grid barrier per iteration, so its partials alternate between two
    // slot groups (8G.. and 11G..): a CTA that runs ahead into the next reduction never
    // overwrites partials a slower CTA is still summing (nor the pre-loop slots 0..2)
    unsigned lep = 0;
    const int bxi = b % RP.ng[0], byi = (b / RP.ng[0]) % RP.ng[1], bzi = b / (RP.ng[0] * RP.ng[1]);
    const int x0 = RP.off[0][bxi], y0 = RP.off[1][byi], z0 = RP.off[2][bzi];
    const int lx = RP.off[0][bxi + 1] - x0, ly = RP.off[1][byi + 1] - y0, lz = RP.off[2][bzi + 1] - z0;
    const int LX = lx + 2, LY = ly + 2, LZ = lz + 2;
    const int H = LX * LY * LZ;
    const int SY = LX, SZ = LX * LY;
    const int nown = lx * ly * lz;
    const int fx = ly * lz, fy = lx * lz, fz = lx * ly;
    const int nface = 2 * (fx + fy + fz);

    // the Gaussian tables live only during phase 0, so they overlay PO (p is first written
    // in iteration 0), extended past it when the tables are longer than the brick
    const int gtab_n = GAUSS ? gauss_smem_len(g) : 0;
    const int extra = gtab_n > nown ? gtab_n - nown : 0;
    double* US = reinterpret_cast<double*>(smem);
    double* RO = US + H;
    double* SO = RO + nown;
    // XG (x in global memory) is a template flag so that the SMEM variant keeps x
    // accesses as shared-memory instructions
    double* XO = XG ? RP.xglob + (size_t)b * RP.xg_stride : SO + nown;
    double* PO = XG ? SO + nown : XO + nown;
    double* tx = PO;
    double* ty = tx + 6 * g.nc[0];
    double* tz = ty + 6 * g.nc[1];
    double* bx_ = tz + 6 * g.nc[2];
    double* by_ = bx_ + g.NX;
    double* bz_ = by_ + g.NY;
    double* RF = PO + nown + extra;
    double* SF = RF + nface;
    int* GID = reinterpret_cast<int*>(SF + nface);
    int* FS = GID + nown;
    int* FG = FS + nface;
    uint8_t* CL = reinterpret_cast<uint8_t*>(FG + nface);

    const int sc = RP.scache ? RP.sc_mode : 0;
    int* SCb = RP.scache ? RP.scache + (size_t)b * RP.sc_stride : nullptr;
    const int nclw = (H + 3) / 4, oFS = nclw, oFG = oFS + nface, oGID = oFG + nface, oOD = oGID + nown;
    build_class_table(T, threadIdx.x, RP.specs ? RP.specs[0].mbase : RP.spec0.mbase, P.cbase, g.dkind);
    if (sc == 2) {
        for (int s = threadIdx.x; s < nclw; s += kResTPB) reinterpret_cast<int*>(CL)[s] = __ldcg(SCb + s);
        for (int s = threadIdx.x; s < H; s += kResTPB) US[s] = 0.0;
    } else {
        for (int s = threadIdx.x; s < H; s += kResTPB) {
            const int u = s % LX, v = (s / LX) % LY, w = s / SZ;
            const int i = x0 + u - 1, j = y0 + v - 1, k = z0 + w - 1;
            const bool in = i >= 0 && i <= g.nc[0] && j >= 0 && j <= g.nc[1] && k >= 0 && k <= g.nc[2];
            CL[s] = in ? (uint8_t)class_of(g, i, j, k) : kNoNode;
            US[s] = 0.0;
        }
    }
    __syncthreads();
    if (sc == 1)
        for (int s = threadIdx.x; s < nclw; s += kResTPB) SCb[s] = reinterpret_cast<const int*>(CL)[s];
    if (prof) RP.prof[120] = global_ns();
    for (int e0 = threadIdx.x; e0 < nface; e0 += kResTPB) {
        if (sc == 2) {
            FS[e0] = __ldcg(SCb + oFS + e0);
            FG[e0] = __ldcg(SCb + oFG + e0);
        } else {
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
            if (sc == 1) {
                SCb[oFS + e0] = FS[e0];
                SCb[oFG + e0] = FG[e0];
            }
        }
        RF[e0] = 0.0;
        SF[e0] = 0.0;
    }
    int od[NPT];
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        const int nl = threadIdx.x + m * kResTPB;
        if (sc == 2) {
            od[m] = __ldcg(SCb + oOD + nl);
            if (nl < nown) {
                GID[nl] = __ldcg(SCb + oGID + nl);
                SO[nl] = 0.0;
                XO[nl] = 0.0;
            }
            continue;
        }
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
            SO[nl] = 0.0;
            XO[nl] = 0.0;
            if (sc == 1) SCb[oGID + nl] = GID[nl];
        }
        if (sc == 1) SCb[oOD + nl] = od[m];
    }

  __shared__ SolveSpec S;                   // this solve's parameters (shared: no registers)
  // MULTI: a solve's residual sums are reduced at the next solve's first grid barrier (one
  // barrier less per solve); its outcome record is written then (thread 0 keeps it here)
  __shared__ SolveInfoDev* pend_info;
  __shared__ int pend_status, pend_it;
  __shared__ double pend_bnorm, pend_rnorm;
  if (threadIdx.x == 0) pend_info = nullptr;
  const int nsp = MULTI ? RP.nspec : 1;
  constexpr int kPS = MULTI ? 1 : 0;        // solve whose phases TLGPU_PROF stamps
  for (int si = 0; si < nsp; ++si) {
    if (MULTI && prof && si == kPS) { np = 0; RP.prof[np++] = global_ns(); }
    __syncthreads();                        // previous solve done with T, PO, US, S
    if (threadIdx.x == 0) S = RP.specs ? RP.specs[si] : RP.spec0;
    __syncthreads();
    const bool gauss = GAUSS && S.src.on;
    build_class_table(T, threadIdx.x, S.mbase, P.cbase, g.dkind);
    if (gauss) build_gauss_tables(g, S.src, tx, ty, tz);
    __syncthreads();
    if (gauss) {
        build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
        __syncthreads();
    }
    if (prof && si == kPS) RP.prof[121] = global_ns();
    auto dvalue = [&](int q) -> double {    // Dirichlet value of this solve
        if (P.gA == nullptr) return P.g_const;
        return __dadd_rn(__dmul_rn(1.0 - S.w, P.gA[q]), __dmul_rn(S.w, P.gB[q]));
    };

    // ---- phase 0: constrained RHS (identical to k_pcg_resident), r0 = b, x = 0 ----
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        const int nl = threadIdx.x + m * kResTPB;
        const int p = GID[nl];
        const int cls = od_cls(od[m]);
        const double told = (!MULTI || S.tin == 0) ? P.T[p] : (S.tin == 1 ? XO[nl] : RP.saved[p]);
        if (MULTI && S.save_before) RP.saved[p] = told;
        XO[nl] = 0.0;                       // x0 = 0
        double bv;
        if (T.nd[cls] == 0.0) {
            bv = dvalue(p);
        } else {
            int i, j, k;
            decode(g, p, i, j, k);
            bv = T.mass[cls] * told;
            if (P.load) bv += P.load[p];
            if (S.load && i >= S.box[0] && i < S.box[1] && j >= S.box[2] && j < S.box[3] && k >= S.box[4] &&
                k < S.box[5])
                bv += S.load[(i - S.box[0]) + (S.box[1] - S.box[0]) * ((j - S.box[2]) + (S.box[3] - S.box[2]) * (k - S.box[4]))];
            if (gauss) bv = add_gaussian(bv, g, tx, ty, tz, bx_, by_, bz_, i, j, k);
            const int sy = g.NX, sz = g.NX * g.NY;
            double lift = 0.0;
            if (i > 0 && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i - 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dvalue(p - 1);
            if (i < g.nc[0] && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * dvalue(p + 1);
            if (j > 0 && T.nd[cls + 3 * (axis_class(j - 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dvalue(p - sy);
            if (j < g.nc[1] && T.nd[cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * dvalue(p + sy);
            if (k > 0 && T.nd[cls + 9 * (axis_class(k - 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dvalue(p - sz);
            if (k < g.nc[2] && T.nd[cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * dvalue(p + sz);
            bv += lift;
        }
        P.b[p] = bv;
        RO[nl] = bv;
        if (od_surf(od[m])) RP.xw[(size_t)g.n + p] = bv;   // xr may still be read (previous tail)
        const double z = __dmul_rn(T.invd[cls], bv);
        acc[0] += bv * bv;
        acc[1] += bv * z;
    }
    if (prof && si == kPS) RP.prof[122] = global_ns();
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) { P.part[0 * G + b] = acc[0]; P.part[1 * G + b] = acc[1]; }
    if (RP.prof && si == kPS && threadIdx.x == 0 && b < 256) RP.prof[512 + b] = global_ns();   // RHS done
    grid.sync();
    {
        const int s2[2] = {0, 1};
        grid_sum_fast<2>(P.part, s2, G, tot);
    }
    if (prof && si == kPS) RP.prof[np++] = global_ns();
    if (MULTI && si > 0 && b == 0 && pend_info) {
        // the previous solve's outcome: its residual partials (slots 4, 5) were published
        // before this solve's first grid barrier
        const int s2[2] = {4, 5};
        grid_sum_fast<2>(P.part, s2, G, tot + 4);
        if (b == 0 && threadIdx.x == 0) {
            int st = pend_status;
            const double tres = pend_bnorm > 0.0 ? sqrt(tot[4]) / pend_bnorm : 0.0;
            if (st == 0 && tot[5] > 0.0) st = 3;
            if (st == 0 && (!isfinite(tres) || tres > 1e2 * P.rtol)) st = 2;
            pend_info->iterations = (st == 1) ? P.maxiter : pend_it;
            pend_info->status = st;
            pend_info->bnorm = pend_bnorm;
            pend_info->rnorm = pend_rnorm;
            pend_info->true_resid = tres;
        }
    }
    const double bb = tot[0];
    double gam = tot[1];                    // r0 . u0
    const double bnorm = sqrt(bb);
    const double atol = P.rtol * bnorm;
    double rnorm = bnorm;
    double rr = bb;
    int it = 0, status = 0;

    double w[NPT];
    double dlt = 0.0;
    if (bb != 0.0) {
        // u0 = M r0 on own + halo (halo r0 from the exchange), w0 = A u0, delta0 = w0.u0
#pragma unroll
        for (int t = 0; t < kResKF; ++t) {
            const int e = threadIdx.x + t * kResTPB;
            if (e < nface && FS[e] >= 0) {
                const double rv = __ldcg(RP.xw + (size_t)g.n + FG[e]);
                RF[e] = rv;
                US[FS[e]] = __dmul_rn(T.invd[CL[FS[e]]], rv);
            }
        }
#pragma unroll
        for (int m = 0; m < NPT; ++m) {
            if (od[m] < 0) continue;
            US[od_s(od[m])] = __dmul_rn(T.invd[od_cls(od[m])], RO[threadIdx.x + m * kResTPB]);
        }
        __syncthreads();
        double d1[1] = {0.0};
#pragma unroll
        for (int m = 0; m < NPT; ++m) {
            if (od[m] < 0) continue;
            const int d = od[m], s = od_s(d), cls = od_cls(d);
            const double uu = US[s];
            const double wv = (T.nd[cls] == 0.0) ? uu : stencil_smem(T, US, s, cls, od_mask(d), SY, SZ);
            w[m] = wv;
            d1[0] += wv * uu;
            if (od_surf(d)) RP.xw[GID[threadIdx.x + m * kResTPB]] = wv;
        }
        block_sum<1>(d1, red);
        if (threadIdx.x == 0) P.part[2 * G + b] = d1[0];
        grid.sync();
        {
            const int s1[1] = {2};
            grid_sum_fast<1>(P.part, s1, G, tot);
        }
        dlt = tot[0];
        double gam_prev = 1.0, alpha_prev = 1.0;
        while (true) {
            rnorm = sqrt(rr);
            // scipy's cg: `for it in range(maxiter): if ||r|| < atol: return ok`, failure when
            // the loop runs out -- the limit is tested before the residual
            if (it >= P.maxiter) { status = 1; break; }
            if (rnorm < atol) { status = 0; break; }
            if (!isfinite(rnorm)) { status = 3; break; }
            const bool first = it == 0;
            const double beta = first ? 0.0 : gam / gam_prev;
            const double alpha = first ? gam / dlt : gam / (dlt - beta * gam / alpha_prev);
            // halo: s = w + beta s, r -= alpha s, u = M r  (w of the halo from the exchange)
#define TL_STAMP(slot) \
    if (prof && si == kPS && it == 3) RP.prof[slot] = global_ns();
            TL_STAMP(100)
            const double* win = RP.xw + (size_t)(it & 1) * g.n;
            double fw[kResKF];
#pragma unroll
            for (int t = 0; t < kResKF; ++t) {
                const int e = threadIdx.x + t * kResTPB;
                fw[t] = (e < nface && FS[e] >= 0) ? __ldcg(win + FG[e]) : 0.0;
            }
            // own: p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s, u = M r
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                if (od[m] < 0) continue;
                const int nl = threadIdx.x + m * kResTPB;
                const int s = od_s(od[m]);
                const double uu = US[s];
                const double pv = first ? uu : __dadd_rn(uu, __dmul_rn(beta, PO[nl]));
                const double sv = first ? w[m] : __dadd_rn(w[m], __dmul_rn(beta, SO[nl]));
                const double rv = __dsub_rn(RO[nl], __dmul_rn(alpha, sv));
                XO[nl] = __dadd_rn(XO[nl], __dmul_rn(alpha, pv));
                PO[nl] = pv;
                SO[nl] = sv;
                RO[nl] = rv;
                // a thread reads and writes only its own nodes' u here (the neighbours' u
                // were last read by the previous stencil, before the grid barrier)
                US[s] = __dmul_rn(T.invd[od_cls(od[m])], rv);
            }
            TL_STAMP(101)
#pragma unroll
            for (int t = 0; t < kResKF; ++t) {
                const int e = threadIdx.x + t * kResTPB;
                if (e >= nface) break;
                const int s = FS[e];
                if (s < 0) continue;
                const double sv = first ? fw[t] : __dadd_rn(fw[t], __dmul_rn(beta, SF[e]));
                const double rv = __dsub_rn(RF[e], __dmul_rn(alpha, sv));
                SF[e] = sv;
                RF[e] = rv;
                US[s] = __dmul_rn(T.invd[CL[s]], rv);
            }
            gam_prev = gam;
            alpha_prev = alpha;
            __syncthreads();
            TL_STAMP(102)
            // w = A u, gamma = r.u, delta = w.u, r.r; publish surface w
            double d3[3] = {0.0, 0.0, 0.0};
            double* wout = RP.xw + (size_t)((it + 1) & 1) * g.n;
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                if (od[m] < 0) continue;
                const int d = od[m], s = od_s(d), cls = od_cls(d), nl = threadIdx.x + m * kResTPB;
                const double uu = US[s];
                const double wv = (T.nd[cls] == 0.0) ? uu : stencil_smem(T, US, s, cls, od_mask(d), SY, SZ);
                w[m] = wv;
                const double rv = RO[nl];
                d3[0] += rv * uu;
                d3[1] += wv * uu;
                d3[2] += rv * rv;
                if (od_surf(d)) wout[GID[nl]] = wv;
            }
            TL_STAMP(103)
            if (RP.bar_count) {
                TL_STAMP(104)
                if (RP.prof && si == kPS && it == 3 && threadIdx.x == 0) RP.prof[256 + b] = global_ns();
                bar_target += (unsigned)G;
                grid_allreduce<3>(d3, red, P.part + (8 + 3 * (lep & 1u)) * G, G, RP.bar_count, bar_target, tot);
                TL_STAMP(105)
                TL_STAMP(106)
            } else {
            double* lp = P.part + (8 + 3 * (lep & 1u)) * G;
            block_sum<3>(d3, red);
            if (threadIdx.x == 0) { lp[0 * G + b] = d3[0]; lp[1 * G + b] = d3[1]; lp[2 * G + b] = d3[2]; }
            TL_STAMP(104)
            if (RP.prof && si == kPS && it == 3 && threadIdx.x == 0) RP.prof[256 + b] = global_ns();   // arrival per CTA
            grid.sync();
            TL_STAMP(105)
            {
                const int s3[3] = {0, 1, 2};
                grid_sum_fast<3>(lp, s3, G, tot);
            }
            TL_STAMP(106)
            }
            ++lep;
#undef TL_STAMP
            if (prof && si == kPS && it < 100) RP.prof[np++] = global_ns();
            gam = tot[0];
            dlt = tot[1];
            rr = tot[2];
            ++it;
        }
    }

    // ---- true residual ||A_c x - b||: publish surface x, gather the halo; x_D = b_D ----
    __syncthreads();                        // all reads of US by the last stencil done
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        const int nl = threadIdx.x + m * kResTPB;
        US[od_s(od[m])] = XO[nl];
        if (od_surf(od[m])) RP.xr[GID[nl]] = XO[nl];
    }
    grid.sync();                            // every CTA's surface x visible
#pragma unroll
    for (int t = 0; t < kResKF; ++t) {
        const int e = threadIdx.x + t * kResTPB;
        if (e < nface && FS[e] >= 0) US[FS[e]] = __ldcg(RP.xr + FG[e]);
    }
    __syncthreads();
    double res[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < NPT; ++m) {
        if (od[m] < 0) continue;
        const int d = od[m], s = od_s(d), cls = od_cls(d);
        const double xp = US[s];
        const double ax = (T.nd[cls] == 0.0) ? xp : stencil_smem(T, US, s, cls, od_mask(d), SY, SZ);
        const int p = GID[threadIdx.x + m * kResTPB];
        const double bv = P.b[p];
        const double dd = ax - bv;
        res[0] += dd * dd;
        res[1] += isfinite(xp) ? 0.0 : 1.0;
        const double xv = (T.nd[cls] == 0.0) ? bv : xp;   // x_D = g = b_D (fem.py:289-290)
        XO[threadIdx.x + m * kResTPB] = xv;
        if (!MULTI || S.tout) P.T[p] = xv;
        if (MULTI && S.snap) S.snap[p] = xv;
    }
    block_sum<2>(res, red);
    bool fin = b == 0;                      // the CTA that writes the outcome record
    if (!MULTI && RP.tail_count) {
        // single solve: the last CTA to finish reduces the residual partials; the others
        // exit without a second grid barrier
        __shared__ bool s_last;
        if (threadIdx.x == 0) {
            P.part[0 * G + b] = res[0];
            P.part[3 * G + b] = res[1];
            __threadfence();
            s_last = atomicAdd(RP.tail_count, 1u) == (unsigned)G - 1;
        }
        __syncthreads();
        if (!s_last) {
            if (prof && si == kPS) { RP.prof[np++] = global_ns(); RP.prof[127] = np; }
            continue;
        }
        __threadfence();
        fin = true;
        if (threadIdx.x == 0) *RP.tail_count = 0;
    } else if (MULTI && si + 1 < nsp) {
        if (threadIdx.x == 0) {
            P.part[4 * G + b] = res[0];
            P.part[5 * G + b] = res[1];
            pend_info = S.info;
            pend_status = status;
            pend_it = it;
            pend_bnorm = bnorm;
            pend_rnorm = rnorm;
        }
        if (prof && si == kPS) { RP.prof[np++] = global_ns(); RP.prof[127] = np; }
        continue;
    } else {
        if (threadIdx.x == 0) { P.part[0 * G + b] = res[0]; P.part[3 * G + b] = res[1]; }
        grid.sync();
    }
    {
        const int s2[2] = {0, 3};
        grid_sum_fast<2>(P.part, s2, G, tot);
    }
    if (fin && threadIdx.x == 0) {
        const double tres = bnorm > 0.0 ? sqrt(tot[0]) / bnorm : 0.0;
        if (status == 0 && tot[1] > 0.0) status = 3;
        if (status == 0 && (!isfinite(tres) || tres > 1e2 * P.rtol)) status = 2;
        S.info->iterations = (status == 1) ? P.maxiter : it;
        S.info->status = status;
        S.info->bnorm = bnorm;
        S.info->rnorm = rnorm;
        S.info->true_resid = tres;
        if (prof && si == kPS) { RP.prof[np++] = global_ns(); RP.prof[127] = np; }
    }
  }
}

// ---------------------------------------------------------------------------------
// Gaussian loads of all solves of a multi-solve launch, computed by one launch before the
// solve so the persistent kernel carries no Gaussian code (registers) and no
// beam-dependent work imbalance.  Values are those add_gaussian evaluates in-kernel; the
// exact cutoff is taken against the floor T_lo instead of the solve's own T_old: for
// T_old >= T_lo / 2 the RHS is bitwise the same (a skipped term has F <= bound <
// 2^-55 m T_lo <= 2^-54 b0, below half an ulp of b0, so b0 + F rounds to b0), and no T_old
// is needed, so all solves fit in one launch.
//
// Only the box of nodes where the term can survive the cutoff is evaluated and stored:
// along each axis, the indices a with 24 mx[a] max(my) max(mz) >= 2^-55 mbase n_min T_lo
// (n_min: the smallest lumped-mass count of a free class; every node outside has
// bound < 2^-55 m T_lo and gets exactly 0).  Every block derives the same box from the
// same tables; block 0 of a solve records it in specs[e].box for the solve kernel.
// grid = (blocks per solve, solves).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gauss_loads(Grid g, SolveSpec* specs, const Gauss* srcs,
                                                     double T_lo, double* loads) {
    extern __shared__ double gtab[];
    __shared__ double massc[27];
    __shared__ double s_thr;
    __shared__ double s_max[3];
    __shared__ int s_lo[3], s_hi[3];
    const int e = blockIdx.y;
    double* out = loads + (size_t)e * g.n;
    double *tx = gtab, *ty = tx + 6 * g.nc[0], *tz = ty + 6 * g.nc[1];
    double *bx_ = tz + 6 * g.nc[2], *by_ = bx_ + g.NX, *bz_ = by_ + g.NY;
    build_gauss_tables(g, srcs[e], tx, ty, tz);
    if (threadIdx.x < 27) {
        int n_p, n_e[3], cnt[3], h0[3], h1[3];
        class_counts(threadIdx.x, n_p, n_e, cnt, h0, h1);
        massc[threadIdx.x] = class_is_dirichlet(threadIdx.x, g.dkind) ? -1.0 : specs[e].mbase * (double)n_p;
    }
    if (threadIdx.x < 3) {
        s_lo[threadIdx.x] = 1 << 30;
        s_hi[threadIdx.x] = -1;
    }
    __syncthreads();
    build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
    if (threadIdx.x == 0) {
        double mmin = 1e300;
        for (int c = 0; c < 27; ++c)
            if (massc[c] > 0.0) mmin = fmin(mmin, massc[c]);
        s_thr = mmin * T_lo * 0x1p-55;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int a = threadIdx.x, n = a == 0 ? g.NX : (a == 1 ? g.NY : g.NZ);
        const double* m = a == 0 ? bx_ : (a == 1 ? by_ : bz_);
        double mx = 0.0;
        for (int i = 0; i < n; ++i) mx = fmax(mx, m[i]);
        s_max[a] = mx;
    }
    __syncthreads();
    {
        const int tot = g.NX + g.NY + g.NZ;
        for (int t = threadIdx.x; t < tot; t += blockDim.x) {
            int a = 0, idx = t;
            if (idx >= g.NX) { idx -= g.NX; a = 1; if (idx >= g.NY) { idx -= g.NY; a = 2; } }
            const double* m = a == 0 ? bx_ : (a == 1 ? by_ : bz_);
            const double other = a == 0 ? s_max[1] * s_max[2] : (a == 1 ? s_max[0] * s_max[2] : s_max[0] * s_max[1]);
            if (24.0 * m[idx] * other >= s_thr) {
                atomicMin(&s_lo[a], idx);
                atomicMax(&s_hi[a], idx + 1);
            }
        }
    }
    __syncthreads();
    int box[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        box[2 * a] = s_hi[a] > s_lo[a] ? s_lo[a] : 0;
        box[2 * a + 1] = s_hi[a] > s_lo[a] ? s_hi[a] : 0;
    }
    if (blockIdx.x == 0 && threadIdx.x < 6) specs[e].box[threadIdx.x] = box[threadIdx.x];
    const int bw = box[1] - box[0], bh = box[3] - box[2], bd = box[5] - box[4];
    const int nb = bw * bh * bd;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nb; q += gridDim.x * blockDim.x) {
        const int i = box[0] + q % bw, j = box[2] + (q / bw) % bh, k = box[4] + q / (bw * bh);
        const double m = massc[class_of(g, i, j, k)];
        if (m < 0.0) { out[q] = 0.0; continue; }
        const double bound = 24.0 * bx_[i] * by_[j] * bz_[k];
        out[q] = (bound < m * T_lo * 0x1p-55) ? 0.0 : gaussian_node_fast(g, tx, ty, tz, i, j, k);
    }
}

}  // namespace tl
