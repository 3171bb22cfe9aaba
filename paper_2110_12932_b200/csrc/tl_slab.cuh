// tl_slab.cuh — z-slab decomposition of the global backward-Euler solve (multi-GPU).
//
// One process per GPU; rank r owns the node planes [k0, k1) of the global grid and
// stores [h0, h1) = [max(k0-1, 0), min(k1+1, NZ)): its own planes plus one halo plane
// per neighbour.  Node planes are contiguous in the reference node order
// (id = i + NX (j + NY k), lpbfsim/mesh.py:406-409), so a halo is one contiguous
// NX*NY run that NCCL send/recv moves without packing.
//
// The solve is the streaming CG of tl_stream.cuh (same sweeps: forward-edge p.Ap in the
// direction sweep, q recomputed in the update sweep) split at its reductions into launches
// the host orchestrates between the collectives:
//   k_slab_rhs        phase 0 over own nodes: b, r = b, x = 0; sums bb, r.z
//   k_slab_direction  p = z (+ beta p) on own AND halo planes (the halo p follows the
//                     same recurrence as its owner, so only r crosses ranks), q = A p
//                     on own nodes; sum p.q
//   k_slab_update     x += alpha p, r -= alpha q (q recomputed); sums r.z, r.r
//   k_slab_residual   ||A x - b||^2 and non-finite count over own nodes
//   k_slab_finish     x_D = b_D
// Every kernel ends with a deterministic two-stage sum: per-block partials, then the
// last block to arrive adds them in block order into sums[].  The host adds the
// ranks' sums in rank order (slab.py), so every rank sees bitwise the same scalars.
// Kernel arrays are base-shifted by the host: a[id] addresses global node id.
#pragma once

#include "tl_stream.cuh"

namespace tl {

constexpr int kSlabTPB = 512;
constexpr int kSlabMaxBlocks = 640;        // partial slots per reduction value

struct SlabParams {
    Grid g;                        // the whole global grid
    double cbase[3], mbase, g_const;
    double *x, *b, *r, *p0, *p1;   // base-shifted: index = global node id
    const double* load;            // base-shifted or nullptr
    Gauss src;
    int own_lo, own_hi;            // owned global ids [own_lo, own_hi)
    int st_lo, st_hi;              // stored global ids [st_lo, st_hi)
    double* part;                  // [4][gridDim] per-block partials
    unsigned* count;               // arrival counter, zero between launches
    double* sums;                  // this rank's totals, 4 slots
};

// Block sum, publish the block partial, and let the last block to arrive add all
// partials in block order (deterministic) into S.sums[slot].
template <int NV>
__device__ __forceinline__ void slab_reduce(const SlabParams& S, const int (&slot)[NV], double (&v)[NV],
                                            double* red) {
    __shared__ int last;
    __shared__ double tot[NV];
    block_sum<NV>(v, red);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) S.part[slot[k] * G + blockIdx.x] = v[k];
        __threadfence();
        last = atomicAdd(S.count, 1u) == (unsigned)(G - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    grid_sum<NV>(S.part, slot, G, tot);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) S.sums[slot[k]] = tot[k];
        *S.count = 0u;
    }
}

template <bool GAUSS>
__global__ void __launch_bounds__(kSlabTPB) k_slab_rhs(SlabParams S) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    extern __shared__ double gtab[];
    const Grid& g = S.g;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    double *tx = gtab, *ty = gtab + 6 * g.nc[0], *tz = ty + 6 * g.nc[1];
    double *bx_ = tz + 6 * g.nc[2], *by_ = bx_ + g.NX, *bz_ = by_ + g.NY;
    if (GAUSS) build_gauss_tables(g, S.src, tx, ty, tz);
    __syncthreads();
    if (GAUSS) {
        build_gauss_bounds(g, tx, ty, tz, bx_, by_, bz_);
        __syncthreads();
    }
    double acc[2] = {0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int p = S.own_lo + blockIdx.x * blockDim.x + threadIdx.x; p < S.own_hi; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        int cls = 13;
        double bv;
        if (!GAUSS && s_free_interior(g, i, j, k)) {
            // class 13, all neighbours free: no lift (the same sum as the general branch)
            bv = T.mass[13] * S.x[p];
            if (S.load) bv += S.load[p];
        } else if (T.nd[cls = class_of(g, i, j, k)] == 0.0) {
            bv = S.g_const;
        } else {
            bv = T.mass[cls] * S.x[p];
            if (S.load) bv += S.load[p];
            if (GAUSS) bv = add_gaussian(bv, g, tx, ty, tz, bx_, by_, bz_, i, j, k);
            // lift, in the order of k_pcg's phase 0 (bitwise the same b)
            const double gc = S.g_const;
            double lift = 0.0;
            if (i > 0 && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i - 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * gc;
            if (i < g.nc[0] && T.nd[cls - axis_class(i, g.nc[0]) + axis_class(i + 1, g.nc[0])] == 0.0) lift += T.c[0][cls] * gc;
            if (j > 0 && T.nd[cls + 3 * (axis_class(j - 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * gc;
            if (j < g.nc[1] && T.nd[cls + 3 * (axis_class(j + 1, g.nc[1]) - axis_class(j, g.nc[1]))] == 0.0) lift += T.c[1][cls] * gc;
            if (k > 0 && T.nd[cls + 9 * (axis_class(k - 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * gc;
            if (k < g.nc[2] && T.nd[cls + 9 * (axis_class(k + 1, g.nc[2]) - axis_class(k, g.nc[2]))] == 0.0) lift += T.c[2][cls] * gc;
            bv += lift;
        }
        S.b[p] = bv;
        S.r[p] = bv;
        S.x[p] = 0.0;
        const double z = __dmul_rn(T.invd[cls], bv);
        acc[0] += bv * bv;
        acc[1] += bv * z;
    }
    const int s[2] = {0, 1};
    slab_reduce<2>(S, s, acc, red);
}

// parity 0: p_old = p0, p_new = p1; parity 1: swapped (k_pcg's ping-pong order)
__global__ void __launch_bounds__(kSlabTPB, 3) k_slab_direction(SlabParams S, int first, double beta,
                                                               int parity) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    const Grid& g = S.g;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    const double* pold = parity ? S.p1 : S.p0;
    double* pnew = parity ? S.p0 : S.p1;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int stride = gridDim.x * blockDim.x;
    // halo planes: the owner's recurrence, pointwise
    const int nlow = S.own_lo - S.st_lo, nhigh = S.st_hi - S.own_hi;
    for (int e = tid; e < nlow + nhigh; e += stride) {
        const int p = e < nlow ? S.st_lo + e : S.own_hi + (e - nlow);
        int i, j, k;
        decode(g, p, i, j, k);
        const double z = __dmul_rn(T.invd[class_of(g, i, j, k)], S.r[p]);
        pnew[p] = first ? z : __dadd_rn(__dmul_rn(beta, pold[p]), z);
    }
    // own nodes: p and p.Ap over the node and its forward edges (the +z edges of the top
    // own plane reach the halo plane, whose p this rank recomputes from r and p_old)
    double pq[1] = {0.0};
    {
        int p = S.own_lo + tid;
        for (; p + stride < S.own_hi; p += 2 * stride) {
            const double a = s_sweep_a_node(g, T, p, S.r, pold, pnew, first != 0, beta);
            const double c = s_sweep_a_node(g, T, p + stride, S.r, pold, pnew, first != 0, beta);
            pq[0] += a;
            pq[0] += c;
        }
        for (; p < S.own_hi; p += stride) pq[0] += s_sweep_a_node(g, T, p, S.r, pold, pnew, first != 0, beta);
    }
    const int s[1] = {2};
    slab_reduce<1>(S, s, pq, red);
}

__global__ void __launch_bounds__(kSlabTPB, 3) k_slab_update(SlabParams S, double alpha, int parity) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    const Grid& g = S.g;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    const double* pnew = parity ? S.p0 : S.p1;
    double a2[2] = {0.0, 0.0};
    {
        const int stride = gridDim.x * blockDim.x;
        int p = S.own_lo + blockIdx.x * blockDim.x + threadIdx.x;
        for (; p + stride < S.own_hi; p += 2 * stride) {
            s_sweep_b_node(g, T, p, S.x, S.r, pnew, alpha, a2[0], a2[1]);
            s_sweep_b_node(g, T, p + stride, S.x, S.r, pnew, alpha, a2[0], a2[1]);
        }
        for (; p < S.own_hi; p += stride) s_sweep_b_node(g, T, p, S.x, S.r, pnew, alpha, a2[0], a2[1]);
    }
    const int s[2] = {0, 1};
    slab_reduce<2>(S, s, a2, red);
}

__global__ void __launch_bounds__(kSlabTPB) k_slab_residual(SlabParams S) {
    __shared__ ClassTable T;
    __shared__ double red[4 * 32];
    const Grid& g = S.g;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    double res[2] = {0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int p = S.own_lo + blockIdx.x * blockDim.x + threadIdx.x; p < S.own_hi; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        const int cls = class_of(g, i, j, k);
        const double xp = S.x[p];
        double ax;
        if (T.nd[cls] == 0.0) ax = xp;
        else ax = apply_free(g, T, p, i, j, k, cls, xp, [&](int q, int) { return S.x[q]; });
        const double d = ax - S.b[p];
        res[0] += d * d;
        res[1] += isfinite(xp) ? 0.0 : 1.0;
    }
    const int s[2] = {0, 3};
    slab_reduce<2>(S, s, res, red);
}

__global__ void __launch_bounds__(kSlabTPB) k_slab_finish(SlabParams S) {
    __shared__ ClassTable T;
    const Grid& g = S.g;
    build_class_table(T, threadIdx.x, S.mbase, S.cbase, g.dkind);
    __syncthreads();
    const int stride = gridDim.x * blockDim.x;
    for (int p = S.own_lo + blockIdx.x * blockDim.x + threadIdx.x; p < S.own_hi; p += stride) {
        int i, j, k;
        decode(g, p, i, j, k);
        if (T.nd[class_of(g, i, j, k)] == 0.0) S.x[p] = S.b[p];
    }
}

}  // namespace tl
