// tl_slabdev.cuh — device-resident CG of the z-slab global solve (multi-GPU data plane).
//
// One process per GPU; rank r owns node planes [k0, k1) of the global grid and stores
// [h0, h1) (one halo plane per neighbour), as tl_slab.cuh.  The solve is scipy's cg
// (lpbfsim/fem.py:271-298) with every scalar decided ON THE DEVICE: the host enqueues
// kernels and collectives and never reads a value inside the CG loop.
//
//   k_sd_begin      control block reset (it = 0, not done)
//   k_slab_rhs      b, r = b, x = 0 on own planes; sums[0] = b.b (= r.r), sums[1] = r.z
//   loop (the host enqueues a predicted number of iterations; surplus ones are no-ops):
//     [all-gather sums -> gath]      every rank's 8 sums, rank order
//     k_sd_dir      prologue: rr, rz = rank-order sums of gath; the stop test of scipy's
//                   loop (||r|| < rtol ||b||, non-finite, maxiter) -> done;
//                   p = z + beta p on the halo planes (the owner's recurrence), then the
//                   bulk-copy z-march sweep A over own planes (tl_tiled.cuh: p, p.Ap over
//                   forward edges); the last CTA sums the item partials -> sums[2]
//     [all-gather]
//     k_sd_upd_flat on the planes a neighbour needs (k0 if r > 0, k1 - 1 if r < world-1):
//                   alpha = rho / sum pq; x += alpha p, r -= alpha A p; block partials
//     [halo exchange of r on the comm stream, overlapped with ...]
//     k_sd_upd      the bulk-copy sweep B over the remaining own planes; the last CTA
//                   adds boundary + item partials in a fixed order -> sums[0] = r.r,
//                   sums[1] = r.z; it += 1
//   [halo x] k_sd_resid (if done): ||A x - b||^2, non-finite count -> sums[3], sums[4]
//   [all-gather] k_sd_finish (if done): the reference's true-residual check (x_D = b_D is
//                   written by k_sd_resid)
//
// Every CTA of every rank computes each scalar from the same gathered values in the same
// order, so all ranks take bitwise the same branch and the iteration count does not
// depend on the collective's reduction algorithm.  Control-block writes are made by the
// last CTA to finish a kernel (after every CTA of that launch has read the block) or by
// CTA 0 for fields no CTA of the launch reads.
#pragma once

#include "tl_slab.cuh"
#include "tl_tiled.cuh"

namespace tl {

constexpr int kSdSums = 8;                 // sums per rank (the all-gather's unit)

struct SlabCtl {
    int it, status, done, maxiter;
    double rtol, bnorm, rnorm, rho, rho_prev, true_resid;
};

struct SlabDev {
    SlabParams S;                  // grid, coefficients, base-shifted arrays, own/stored ids
    int k0, k1;                    // owned planes
    int world;
    const double* gath;            // [world][kSdSums]
    SlabCtl* ctl;
    double* ipart;                 // item partials of the tiled sweeps (3 * kTMaxItems)
    double* bpart;                 // block partials of the flat boundary sweep (2 * kSlabMaxBlocks)
    unsigned* icount;              // arrival counter of the tiled sweeps (zero between launches)
    unsigned* ictr;                // item counter of the tiled sweeps (zero between launches)
    int nbnd;                      // blocks of the boundary sweep that wrote bpart (0: none)
};

__device__ __forceinline__ double sd_gsum(const SlabDev& D, int slot) {
    double s = 0.0;
    for (int r = 0; r < D.world; ++r) s += __ldcg(D.gath + r * kSdSums + slot);
    return s;
}

__global__ void k_sd_begin(SlabCtl* ctl, double rtol, int maxiter) {
    ctl->it = 0;
    ctl->status = 0;
    ctl->done = 0;
    ctl->maxiter = maxiter;
    ctl->rtol = rtol;
    ctl->bnorm = 0.0;
    ctl->rnorm = 0.0;
    ctl->rho = 0.0;
    ctl->rho_prev = 1.0;
    ctl->true_resid = 0.0;
}

// Last CTA of a non-cooperative launch: returns true in every thread of that CTA, after a
// fence that makes the other CTAs' partials visible.
__device__ __forceinline__ bool sd_last_cta(unsigned* count) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// ---- direction: stop test, halo p, bulk-copy sweep A over own planes --------------------
template <int NCW, int NPT>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_sd_dir(SlabDev D, TPlan tp) {
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    __shared__ double ired[2][32];
    __shared__ __align__(8) uint64_t full[kTMaxStages], empty[kTMaxStages];
    __shared__ int s_item[kTMaxStages];
    const SlabParams& S = D.S;
    const Grid& g = S.g;
    if (__ldcg(&D.ctl->done)) return;
    const int it = __ldcg(&D.ctl->it);
    const double rr = sd_gsum(D, 0), rz = sd_gsum(D, 1);
    const double bnorm = it == 0 ? sqrt(rr) : __ldcg(&D.ctl->bnorm);   // r0 = b
    const double rnorm = sqrt(rr);
    const double rtol = __ldcg(&D.ctl->rtol);
    int status = -1;
    if (it == 0 && rr == 0.0) status = 0;                 // b = 0: x = 0 (fem.py:275-276)
    else if (it >= __ldcg(&D.ctl->maxiter)) status = 1;   // scipy: the limit before the residual
    else if (rnorm < rtol * bnorm) status = 0;
    else if (!isfinite(rnorm)) status = 3;
    if (status >= 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            D.ctl->status = status;
            D.ctl->rnorm = rnorm;
            if (it == 0) D.ctl->bnorm = bnorm;
            D.ctl->done = 1;
        }
        return;
    }
    const double rho = rz;
    const double beta = it > 0 ? rho / __ldcg(&D.ctl->rho_prev) : 0.0;
    const bool first = it == 0;
    const double* pold = (it & 1) ? S.p1 : S.p0;
    double* pnew = (it & 1) ? S.p0 : S.p1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < tp.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    if (tp.I > 0) t_zero_ring(tp, t_sm);
    __syncthreads();
    const bool producer = (threadIdx.x >> 5) == NCW;
    uint32_t t = 0;
    if (producer) {
        if ((threadIdx.x & 31) == 0)
            t_produce<false>(g, tp, t_sm, full, empty, s_item, D.ictr, t, first, S.r, pold, nullptr, nullptr);
    } else {
        // halo planes: p by the owner's recurrence, pointwise (own planes: the sweep below)
        const int nlow = S.own_lo - S.st_lo, nhigh = S.st_hi - S.own_hi;
        const int nt = NCW * 32;
        for (int e = blockIdx.x * nt + threadIdx.x; e < nlow + nhigh; e += gridDim.x * nt) {
            const int p = e < nlow ? S.st_lo + e : S.own_hi + (e - nlow);
            int i, j, k;
            decode(g, p, i, j, k);
            const double z = __dmul_rn(T.invd[class_of(g, i, j, k)], S.r[p]);
            pnew[p] = first ? z : __dadd_rn(__dmul_rn(beta, pold[p]), z);
        }
        t_consume_a<NCW, NPT>(g, tp, T, full, empty, s_item, t, first, beta, pnew, D.ipart, ired);
    }
    if (sd_last_cta(D.icount)) {
        t_grid_sum<1>(D.ipart, tp.I, red, tot);
        if (threadIdx.x == 0) {
            S.sums[2] = tot[0];
            D.ctl->rho = rho;
            if (it == 0) D.ctl->bnorm = bnorm;
            *D.icount = 0u;
            *D.ictr = 0u;
        }
    }
}

// ---- update, boundary planes: flat sweep over planes [zlo, zhi) (one or two planes) ------
// Writes its block partials to D.bpart (slots 0: r.z, 1: r.r); the tiled update that
// follows adds them in block order ahead of its item partials.
__global__ void __launch_bounds__(kSlabTPB, 2) k_sd_upd_flat(SlabDev D, int zlo0, int zhi0, int zlo1, int zhi1) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    const SlabParams& S = D.S;
    const Grid& g = S.g;
    if (__ldcg(&D.ctl->done)) return;
    const int it = __ldcg(&D.ctl->it);
    const double alpha = __ldcg(&D.ctl->rho) / sd_gsum(D, 2);
    const double* pnew = (it & 1) ? S.p0 : S.p1;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    const int nxy = g.NX * g.NY;
    const int n0 = (zhi0 - zlo0) * nxy, n1 = (zhi1 - zlo1) * nxy;
    double a2[2] = {0.0, 0.0};
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n0 + n1; e += gridDim.x * blockDim.x) {
        const int p = e < n0 ? zlo0 * nxy + e : zlo1 * nxy + (e - n0);
        s_sweep_b_node(g, T, p, S.x, S.r, pnew, alpha, a2[1], a2[0]);
    }
    block_sum<2>(a2, red);
    if (threadIdx.x == 0) {
        D.bpart[blockIdx.x] = a2[0];
        D.bpart[kSlabMaxBlocks + blockIdx.x] = a2[1];
    }
}

// ---- update, interior: the bulk-copy sweep B over own planes minus the boundary ----------
template <int NCW, int NPT>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_sd_upd(SlabDev D, TPlan tp) {
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    __shared__ double ired[2][32];
    __shared__ __align__(8) uint64_t full[kTMaxStages], empty[kTMaxStages];
    __shared__ int s_item[kTMaxStages];
    const SlabParams& S = D.S;
    const Grid& g = S.g;
    if (__ldcg(&D.ctl->done)) return;
    const int it = __ldcg(&D.ctl->it);
    const double rho = __ldcg(&D.ctl->rho);
    const double alpha = rho / sd_gsum(D, 2);
    const double* pnew = (it & 1) ? S.p0 : S.p1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < tp.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    if (tp.I > 0) t_zero_ring(tp, t_sm);
    __syncthreads();
    const bool producer = (threadIdx.x >> 5) == NCW;
    uint32_t t = 0;
    if (tp.I > 0) {
        if (producer) {
            if ((threadIdx.x & 31) == 0)
                t_produce<true>(g, tp, t_sm, full, empty, s_item, D.ictr, t, false, S.r, nullptr, pnew, S.x,
                                tp.snake != 0);
        } else {
            // item partials: slot 0 r.z, slot 1 r.r (t_consume_b's order)
            t_consume_b<NCW, NPT>(g, tp, T, full, empty, s_item, t, alpha, false, S.x, S.r, D.ipart, ired);
        }
    }
    if (sd_last_cta(D.icount)) {
        // fixed order: boundary block partials (block order), then the item partials
        double s2[2] = {0.0, 0.0};
        for (int b = threadIdx.x; b < D.nbnd; b += blockDim.x) {
            s2[0] += __ldcg(D.bpart + kSlabMaxBlocks + b);      // r.z
            s2[1] += __ldcg(D.bpart + b);                       // r.r
        }
        block_sum<2>(s2, red);
        if (threadIdx.x == 0) { tot[0] = s2[0]; tot[1] = s2[1]; }
        __syncthreads();
        const double bz = tot[0], br = tot[1];
        __syncthreads();
        double it2[2];
        if (tp.I > 0) {
            t_grid_sum<2>(D.ipart, tp.I, red, tot);
            it2[0] = tot[0];
            it2[1] = tot[1];
        } else {
            it2[0] = it2[1] = 0.0;
        }
        if (threadIdx.x == 0) {
            S.sums[1] = bz + it2[0];           // r.z
            S.sums[0] = br + it2[1];           // r.r
            D.ctl->rho_prev = rho;
            D.ctl->it = it + 1;
            *D.icount = 0u;
            *D.ictr = 0u;
        }
    }
}

// ---- after the loop (no-ops until the stop test fired) ----------------------------------
__global__ void __launch_bounds__(kSlabTPB) k_sd_resid(SlabDev D) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    const SlabParams& S = D.S;
    const Grid& g = S.g;
    if (!__ldcg(&D.ctl->done)) return;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    double res[2] = {0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    // s_resid_node: interior fast path; also re-imposes x_D = b_D (fem.py:289-290) after the
    // node's own term (neighbours read x_D with weight 0, so either value gives the same sum)
    for (int p = S.own_lo + blockIdx.x * blockDim.x + threadIdx.x; p < S.own_hi; p += stride)
        s_resid_node(g, T, p, S.x, S.b, res);
    const int s[2] = {3, 4};
    slab_reduce<2>(S, s, res, red);
}

__global__ void __launch_bounds__(kSlabTPB) k_sd_finish(SlabDev D) {
    if (!__ldcg(&D.ctl->done)) return;
    // (x_D = b_D was written by k_sd_resid)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // the reference's post-check (fem.py:286-288) and FieldState's finite check
        const double bnorm = D.ctl->bnorm;
        const double tres = bnorm > 0.0 ? sqrt(sd_gsum(D, 3)) / bnorm : 0.0;
        int st = D.ctl->status;
        if (st == 0 && sd_gsum(D, 4) > 0.0) st = 3;
        if (st == 0 && (!isfinite(tres) || tres > 1e2 * D.ctl->rtol)) st = 2;
        D.ctl->status = st;
        D.ctl->true_resid = tres;
        D.ctl->done = 2;                      // finished (the host polls for 2)
    }
}

}  // namespace tl
