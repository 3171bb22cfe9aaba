// tl_tiled.cuh — z-marching CG loop fed by the bulk-copy engine (sm_100a, fp64).
//
// Same iterations as k_s_cg (tl_stream.cuh; scipy's cg as used by lpbfsim/fem.py:271-298)
// and the same per-node arithmetic (s_sweep_a_node / s_sweep_b_node read through a
// shared-memory view instead of global memory), so a node's p, x, r are bitwise the ones
// k_s_cg computes for the same alpha and beta.
//
// Why: the flat grid-stride sweeps of k_s_cg fetch each node's y and z neighbours from L2
// (3x the DRAM bytes of the operand in sweep A, 5x in sweep B), and the L2 slice
// throughput (~6.3 kB/clk chip-wide, B300_MICROARCH.md) caps them below the HBM peak.
// Here every operand plane crosses L2 once per item:
//
//   item      = (row block jb: H full x-rows, z chunk kc: planes [k0, k1))
//   stage     = one z-plane of an item: the item's rows (plus one halo row on each side
//               for the stencil operand) of each vector, ONE contiguous range per vector
//               (full x-rows are contiguous in the reference node order), moved by
//               cp.async.bulk into a ring of NS shared-memory stages
//   producer  = one lane of the last warp: takes items from a per-sweep atomic counter
//               (dynamic balance), waits for a free stage (empty mbarrier), arms the full
//               mbarrier with the byte count and issues the bulk copies
//   consumers = NCW warps: wait for plane k (and k+1, and keep k-1), compute the plane,
//               release the stage; no CTA-wide barrier in the march
//
// Sweep A (p = z + beta p_old and p.Ap over forward edges) needs r and p_old at planes
// k, k+1 and rows j0..j1 (one forward halo row); sweep B (q = A p, x += alpha p,
// r -= alpha q) needs p at planes k-1, k, k+1 with one halo row each side, and x, r at
// plane k.  Dot products are reduced per item in a fixed order and the item partials
// summed in item order by every CTA after the grid barrier: the result does not depend
// on which CTA ran which item (deterministic despite the dynamic schedule).
//
// Snake order (TPlan::snake): sweep A walks the items bottom-up, sweep B top-down.  On
// grids of a few L2 sizes (cfg4 local, cfg3 global: ~50 MB per vector against 126 MB of
// L2) a sweep then starts on the planes the previous sweep read and wrote last, which are
// still in L2 (p and r for sweep B; r and p_old for the next sweep A).
#pragma once

#include "tl_stream.cuh"

namespace tl {

constexpr int kTMaxStages = 16;
constexpr int kTMaxChunks = 96;            // z chunks (guided: large first, small last)
constexpr int kTPartItems = 4096;          // offset of the item partials in PcgParams::part
constexpr int kTMaxItems = 16384;          // sweep A: slot 0, sweep B: slots 1, 2 (3 * kTMaxItems)
constexpr int kTCounter = 2048;            // offset (in doubles) of the 4 sweep counters

struct TPlan {
    int H;          // rows per item
    int NB;         // row blocks
    int C;          // z chunks
    int I;          // items = NB * C
    int NS;         // ring stages
    int stage;      // doubles per stage
    int RA;         // sweep A: r at [0, RA), p_old at [RA, 2 RA)
    int RB, RX;     // sweep B: p at [0, RB), x at [RB, RB + RX), r at [RB + RX, RB + 2 RX)
    FastDiv nsd, nbd;       // division by NS, NB
    int ncw;        // consumer warps of the kernel instance this plan is for (host side)
    FastDiv iid;    // division by I (batched solves: global item = system * I + item)
    int snake;      // 1: sweep B takes the items from the top of the grid down (L2 reuse, below)
    unsigned long long* prof;    // TLGPU_PROF=1: %globaltimer stamps of iteration 3, slot 1024 + 16 CTA + e
    short kb[kTMaxChunks + 1];   // chunk kc = planes [kb[kc], kb[kc + 1])
};

// Ring slot of position u; parity of its phase in *ph.
__device__ __forceinline__ int t_slot(const TPlan& tp, uint32_t u, unsigned& ph) {
    const uint32_t q = tp.nsd.div(u);
    ph = q & 1u;
    return (int)(u - q * (uint32_t)tp.NS);
}
__device__ __forceinline__ int t_slot(const TPlan& tp, uint32_t u) {
    unsigned ph;
    return t_slot(tp, u, ph);
}

// ---- mbarrier / bulk-copy primitives (PTX ISA 8.0+, sm_90+) -------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    unsigned done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// Global -> shared bulk copy completing on mbarrier b (16-byte aligned, bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ unsigned long long t_ns() { return timer_ns(); }
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Zero the ring once per launch (all threads; the caller's next CTA barrier orders it
// before the first bulk copy): the lean plane loops read words no copy ever writes
// (rows outside the grid) under a zero coupling, so those words must be finite.
__device__ __forceinline__ void t_zero_ring(const TPlan& tp, double* sm) {
    const int n = tp.NS * tp.stage;
    for (int e = threadIdx.x; e < n; e += blockDim.x) sm[e] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Batched solves (BASELINE config 5: many scenarios on grids of one shape): B independent
// systems advance in lockstep through one sweep; the global item id is system * I + item,
// a finished system's items are skipped, and each item takes its arrays, coefficients and
// scalars from its system.
constexpr int kTBMax = 64;                 // systems per batched launch
struct TBatchCtx {
    const PcgParams* Ps;                   // the systems (device memory; one grid shape)
    const int* done;                       // per system: finished (shared memory)
    const double* alpha;                   // per-system scalars of this iteration (shared memory)
    const double* beta;
    int B;
    int parity;                            // iteration parity: p_old = parity ? p1 : p0
    int light0;                            // first iteration: r0 = b, x0 = 0 implied
};

// Item geometry.
struct TItem {
    int j0, j1, k0, k1;
};
__device__ __forceinline__ TItem t_item(const Grid& g, const TPlan& tp, int item) {
    const int kc = (int)tp.nbd.div((uint32_t)item), jb = item - kc * tp.NB;
    TItem it;
    it.j0 = jb * tp.H;
    it.j1 = min(g.NY, it.j0 + tp.H);
    it.k0 = tp.kb[kc];
    it.k1 = tp.kb[kc + 1];
    return it;
}
// Aligned (even) start of the node range [a, b) and its byte count rounded up to 16.
__device__ __forceinline__ int t_abeg(int a) { return a & ~1; }
__device__ __forceinline__ unsigned t_bytes(int a, int b) { return (unsigned)((((b + 1) & ~1) - (a & ~1)) * 8); }

// ---- producer ---------------------------------------------------------------------------
// Sweep A stage of plane k: r, p_old rows [j0, min(j1 + 1, NY)); sweep B stage of plane k:
// p rows [max(j0 - 1, 0), min(j1 + 1, NY)), plus x, r rows [j0, j1) on centre planes
// (x == nullptr: x = 0, not loaded).
template <bool SWEEP_B, bool BATCH = false>
__device__ void t_produce(const Grid& g, const TPlan& tp, double* sm, uint64_t* full, uint64_t* empty,
                          int* s_item, unsigned* ctr, uint32_t& t, bool first, const double* r,
                          const double* pold, const double* pc, const double* x, bool rev = false,
                          const TBatchCtx* bc = nullptr) {
    const int NXY = g.NX * g.NY;
    const int Itot = BATCH ? bc->B * tp.I : tp.I;
    // the first item of every CTA is static (no counter round trip at the sweep start);
    // the rest come from the counter, offset by the grid size
    unsigned next = blockIdx.x;
    while (true) {
        if ((int)next >= Itot) {
            unsigned ph;
            const int s = t_slot(tp, t, ph);
            mbar_wait(&empty[s], ph ^ 1);
            s_item[s] = -1;
            mbar_arrive(&full[s]);
            ++t;
            return;
        }
        // rev: the sweep walks the items from the last one down, so it starts on the planes
        // the previous sweep touched last (still in L2)
        const int gitem = rev ? Itot - 1 - (int)next : (int)next;
        next = gridDim.x + atomicAdd(ctr, 1u);   // the next item's id arrives while this one streams
        int item = gitem;
        if (BATCH) {
            const int sy_ = (int)tp.iid.div((uint32_t)gitem);
            item = gitem - sy_ * tp.I;
            if (bc->done[sy_]) continue;
            const PcgParams& Q = bc->Ps[sy_];
            r = bc->light0 ? Q.b : Q.r;
            pold = bc->parity ? Q.p1 : Q.p0;
            pc = bc->parity ? Q.p0 : Q.p1;
            x = bc->light0 ? nullptr : Q.T;
        }
        const TItem it = t_item(g, tp, item);
        const int ks = SWEEP_B ? max(it.k0 - 1, 0) : it.k0;
        const int ke = min(it.k1, g.NZ - 1);
        for (int k = ks; k <= ke; ++k) {
            unsigned ph;
            const int s = t_slot(tp, t, ph);
            mbar_wait(&empty[s], ph ^ 1);
            if (k == ks) s_item[s] = gitem;
            double* st = sm + (size_t)s * tp.stage;
            if (!SWEEP_B) {
                const int a = k * NXY + it.j0 * g.NX, b = k * NXY + min(it.j1 + 1, g.NY) * g.NX;
                const unsigned nb = t_bytes(a, b);
                mbar_arrive_tx(&full[s], first ? nb : 2 * nb);
                bulk_g2s(st, r + t_abeg(a), nb, &full[s]);
                if (!first) bulk_g2s(st + tp.RA, pold + t_abeg(a), nb, &full[s]);
            } else {
                const int a = k * NXY + max(it.j0 - 1, 0) * g.NX, b = k * NXY + min(it.j1 + 1, g.NY) * g.NX;
                const unsigned nb = t_bytes(a, b);
                const bool centre = k >= it.k0 && k < it.k1;
                const int c = k * NXY + it.j0 * g.NX, d = k * NXY + it.j1 * g.NX;
                const unsigned nc = centre ? t_bytes(c, d) : 0u;
                mbar_arrive_tx(&full[s], nb + (x ? 2 : 1) * nc);
                // the stage starts at row j0 - 1 even where that row does not exist (j0 = 0)
                bulk_g2s(st + (t_abeg(a) - t_abeg(k * NXY + (it.j0 - 1) * g.NX)), pc + t_abeg(a), nb, &full[s]);
                if (centre) {
                    if (x) bulk_g2s(st + tp.RB, x + t_abeg(c), nc, &full[s]);
                    bulk_g2s(st + tp.RB + tp.RX, r + t_abeg(c), nc, &full[s]);
                }
            }
            ++t;
        }
    }
}

// Ring cursor: position t, its slot and phase parity, advanced without divisions.
struct TRing {
    uint32_t t;
    int s;
    unsigned ph;
    __device__ __forceinline__ void set(const TPlan& tp, uint32_t u) {
        t = u;
        s = t_slot(tp, u, ph);
    }
    __device__ __forceinline__ void adv(const TPlan& tp) {
        ++t;
        if (++s == tp.NS) { s = 0; ph ^= 1u; }
    }
    __device__ __forceinline__ TRing next(const TPlan& tp) const {
        TRing r = *this;
        r.adv(tp);
        return r;
    }
};
// Consumer-side release of a stage (one arrival per warp) and wait for a full stage.
__device__ __forceinline__ void t_release(uint64_t* empty, const TRing& r) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[r.s]);
}
__device__ __forceinline__ void t_wait_full(uint64_t* full, const TRing& r) { mbar_wait(&full[r.s], r.ph); }

// Per-item fixed-order reduction of NV values over the NCW consumer warps; warp 0 lane 0
// writes part[v * I + item].
template <int NV, int NCW>
__device__ __forceinline__ void t_item_sum(double (&v)[NV], double (*ired)[32], double* part, int I, int item) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) ired[k][w] = v[k];
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < NCW; ++u) s += ired[k][u];
            part[k * I + item] = s;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
}

// The ring lives in dynamic shared memory; helpers index it through this symbol so that
// every access compiles to LDS.
extern __shared__ __align__(128) double t_sm[];

// Sweep A value of p at node q (plane offset o: t_sm[o + q] = r[q], t_sm[o + RA + q] = p_old[q]).
__device__ __forceinline__ double t_pv(int o, int RA, int q, double iv, bool first, double beta) {
    const double z = __dmul_rn(iv, t_sm[o + q]);
    return first ? z : __dadd_rn(__dmul_rn(beta, t_sm[o + RA + q]), z);
}

// Shared-memory load by 32-bit shared address: the lean plane loops address the ring from
// one base register (generic indexing of the extern array costs a shared-window
// computation per access).  volatile: never hoisted above the mbarrier waits.
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// Sweep A value of p from the stage words at shared address a (r) and a + ra8 (p_old).
__device__ __forceinline__ double t_pva(uint32_t a, uint32_t ra8, double iv, bool first, double beta) {
    const double z = __dmul_rn(iv, lds64(a));
    return first ? z : __dadd_rn(__dmul_rn(beta, lds64(a + ra8)), z);
}
// Same after the first iteration: p = beta p_old + z.
__device__ __forceinline__ double t_pvb(uint32_t a, uint32_t ra8, double iv, double beta) {
    return __dadd_rn(__dmul_rn(beta, lds64(a + ra8)), __dmul_rn(iv, lds64(a)));
}

// Per-item node table of a consumer thread: node m of every plane of the item sits at
// offset off[m] inside the plane, with its x/y class part cxy[m] = cx + 3 cy, the class
// steps to its x+ / y+ neighbours and flag bits (below).  Every node then runs the same
// branch-free code: no warp of the CTA is slowed by boundary nodes (the empty barrier of
// a stage waits for the slowest warp).
enum : unsigned { kFOk = 1, kFXm = 2, kFXp = 4, kFYm = 8, kFYp = 16, kFCol = 32 };
template <int NPT, int NT>
struct TNodes {
    int off[NPT], cxy[NPT], dxp[NPT], dyp[NPT];
    unsigned fl[NPT];
    __device__ __forceinline__ void init(const Grid& g, const TItem& it) {
        const int nn = (it.j1 - it.j0) * g.NX;
        // free (non-Dirichlet) node of x/y classes (a, b) on a plane with cz >= 1
        auto freec = [&](int a, int b) { return !class_is_dirichlet(a + 3 * b + 9, g.dkind); };
#pragma unroll
        for (int m = 0; m < NPT; ++m) {
            const int e0 = threadIdx.x + m * NT;
            const int e = e0 < nn ? e0 : 0;     // no node: addresses of the item's first node, flags 0
            const int jj = (int)g.divX.div((uint32_t)e);
            const int i = e - jj * g.NX, j = it.j0 + jj;
            off[m] = i + g.NX * j;
            const int cx = axis_class(i, g.nc[0]), cy = axis_class(j, g.nc[1]);
            cxy[m] = cx + 3 * cy;
            const int cxn = i < g.nc[0] ? axis_class(i + 1, g.nc[0]) : cx;
            const int cyn = j < g.nc[1] ? axis_class(j + 1, g.nc[1]) : cy;
            dxp[m] = cxn - cx;
            dyp[m] = 3 * (cyn - cy);
            unsigned f = e0 < nn ? kFOk : 0u;
            if (i > 0 && freec(axis_class(i - 1, g.nc[0]), cy)) f |= kFXm;
            if (i < g.nc[0] && freec(cxn, cy)) f |= kFXp;
            if (j > 0 && freec(cx, axis_class(j - 1, g.nc[1]))) f |= kFYm;
            if (j < g.nc[1] && freec(cx, cyn)) f |= kFYp;
            if (freec(cx, cy)) f |= kFCol;
            fl[m] = f;
            // keep the table in registers: without this the compiler recomputes the
            // division by NX inside the plane loops to save registers
            asm volatile("" : "+r"(off[m]), "+r"(fl[m]));
        }
    }
};

// ---- consumers: sweep A ------------------------------------------------------------------
// p = z (+ beta p_old) and its p.Ap contribution over the node and its free forward
// neighbours (s_sweep_a_node, one expression for every class).
// Batched consumers: the item's system selects the arrays, the scalars and the class table
// (rebuilt in shared memory when the system changes; every consumer warp walks the same
// item sequence, so the named barriers around the rebuild are uniform).
template <int NCW>
__device__ __forceinline__ void t_batch_table(const Grid& g, ClassTable& T, const PcgParams& Q) {
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    build_class_table(T, threadIdx.x, Q.mbase, Q.cbase, g.dkind);
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
}

template <int NCW, int NPT, bool BATCH = false>
__device__ void t_consume_a(const Grid& g, const TPlan& tp, ClassTable& T, uint64_t* full, uint64_t* empty,
                            const int* s_item, uint32_t& t, bool first, double beta, double* __restrict__ pnew,
                            double* part, double (*ired)[32], unsigned long long* pf = nullptr,
                            const TBatchCtx* bc = nullptr) {
    const int NXY = g.NX * g.NY, sy = g.NX, RA = tp.RA;
    constexpr int NT = NCW * 32;
    int cur_sys = -1;
    TRing cur;
    cur.set(tp, t);
    while (true) {
        t_wait_full(full, cur);
        if (pf && threadIdx.x == 0) { *pf = t_ns(); pf = nullptr; }      // first stage of the sweep landed
        int item = s_item[cur.s];
        if (item < 0) { t_release(empty, cur); cur.adv(tp); t = cur.t; return; }
        if (BATCH) {
            const int sy_ = (int)tp.iid.div((uint32_t)item);
            item -= sy_ * tp.I;
            const PcgParams& Q = bc->Ps[sy_];
            if (sy_ != cur_sys) { t_batch_table<NCW>(g, T, Q); cur_sys = sy_; }
            pnew = bc->parity ? Q.p0 : Q.p1;
            beta = bc->beta[sy_];
            part = Q.part + kTPartItems;
        }
        const TItem it = t_item(g, tp, item);
        TNodes<NPT, NT> nd;
        nd.init(g, it);
        // Lean planes (1 <= k <= NZ - 3: the node and its z+ neighbour have z class 1; not
        // the first iteration): the node's coefficients are item constants held in
        // registers, with absent or Dirichlet forward neighbours folded in as zero
        // couplings, identity rows as diag = 1 (a = pp * pp) and threads without a node as
        // all-zero coefficients.  Every load is unconditional: an absent neighbour's
        // address holds either another node's value or ring words the kernel zeroed at
        // its start (finite either way), times a zero coupling.  The node's own p is the
        // z+ value computed on the previous plane (same class, same operations).
        double ivo[NPT], ivx[NPT], ivy[NPT], dg[NPT], ex[NPT], ey[NPT], ez[NPT], carry[NPT];
        constexpr bool kLean = NPT <= 2;
        if (kLean) {
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                const int cl = nd.cxy[m] + 9;
                const unsigned f = nd.fl[m];
                const bool ok = f & kFOk;
                const bool cpl = ok && T.nd[cl] != 0.0;
                ivo[m] = T.invd[cl];
                ivx[m] = T.invd[cl + nd.dxp[m]];
                ivy[m] = T.invd[cl + nd.dyp[m]];
                dg[m] = ok ? T.diag[cl] : 0.0;
                ex[m] = (cpl && (f & kFXp)) ? T.c[0][cl] : 0.0;
                ey[m] = (cpl && (f & kFYp)) ? T.c[1][cl] : 0.0;
                ez[m] = (cpl && (f & kFCol)) ? T.c[2][cl] : 0.0;
                carry[m] = 0.0;
            }
        }
        bool have = false;                       // carry holds this plane's own p
        uint32_t sm0 = smem_u32(t_sm);
        uint32_t ra8 = 8u * (uint32_t)RA, sy8 = 8u * (uint32_t)sy;
        asm volatile("" : "+r"(sm0), "+r"(ra8), "+r"(sy8));      // computed once per item
        double acc[1] = {0.0};
        for (int k = it.k0; k < it.k1; ++k) {
            const bool nxt = k + 1 < g.NZ;
            const TRing nx = cur.next(tp);
            if (nxt) t_wait_full(full, nx);
            const int kb = k * NXY;
            const int s0 = cur.s * tp.stage - t_abeg(kb + it.j0 * g.NX);
            const int o1 = nxt ? nx.s * tp.stage - t_abeg(kb + NXY + it.j0 * g.NX) : 0;
            if (kLean && !first && k >= 1 && k <= g.NZ - 3) {
                const uint32_t b0 = sm0 + 8u * (uint32_t)(s0 + kb), b1 = sm0 + 8u * (uint32_t)(o1 + kb + NXY);
#pragma unroll
                for (int m = 0; m < NPT; ++m) {
                    const uint32_t a0 = b0 + 8u * (uint32_t)nd.off[m];
                    const double pz = t_pvb(b1 + 8u * (uint32_t)nd.off[m], ra8, ivo[m], beta);
                    const double pp = have ? carry[m] : t_pvb(a0, ra8, ivo[m], beta);
                    const double px = t_pvb(a0 + 8u, ra8, ivx[m], beta);
                    const double py = t_pvb(a0 + sy8, ra8, ivy[m], beta);
                    if (nd.fl[m] & kFOk) pnew[kb + nd.off[m]] = pp;
                    acc[0] += pp * (dg[m] * pp - 2.0 * ((ex[m] * px + ey[m] * py) + ez[m] * pz));
                    carry[m] = pz;
                }
                have = true;
            } else {
            have = false;
            const int cz = axis_class(k, g.nc[2]);
            const int dzp = nxt ? 9 * (axis_class(k + 1, g.nc[2]) - cz) : 0;
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                const unsigned f = nd.fl[m];
                if (!(f & kFOk)) continue;
                const int p = kb + nd.off[m];
                const int cl = nd.cxy[m] + 9 * cz;
                const double pp = t_pv(s0, RA, p, T.invd[cl], first, beta);
                pnew[p] = pp;
                double a;
                if (T.nd[cl] == 0.0) {
                    a = pp * pp;                         // identity row
                } else {
                    const double px = (f & kFXp) ? t_pv(s0, RA, p + 1, T.invd[cl + nd.dxp[m]], first, beta) : 0.0;
                    const double py = (f & kFYp) ? t_pv(s0, RA, p + sy, T.invd[cl + nd.dyp[m]], first, beta) : 0.0;
                    const double pz = (nxt && (f & kFCol)) ? t_pv(o1, RA, p + NXY, T.invd[cl + dzp], first, beta) : 0.0;
                    a = pp * (T.diag[cl] * pp - 2.0 * ((T.c[0][cl] * px + T.c[1][cl] * py) + T.c[2][cl] * pz));
                }
                acc[0] += a;
            }
            }
            t_release(empty, cur);
            cur.adv(tp);
        }
        if (it.k1 < g.NZ) { t_release(empty, cur); cur.adv(tp); }    // the forward plane k1
        t_item_sum<1, NCW>(acc, ired, part, tp.I, item);
        t = cur.t;
    }
}

// ---- consumers: sweep B ------------------------------------------------------------------
// q = A_c p (apply_free, one expression for every class), x += alpha p, r -= alpha q.
// Holds stages k and k+1; the p values of plane k-1 at the thread's own nodes (its z
// neighbour below) are the centre values of the previous plane, kept in registers.
template <int NCW, int NPT, bool BATCH = false>
__device__ void t_consume_b(const Grid& g, const TPlan& tp, ClassTable& T, uint64_t* full, uint64_t* empty,
                            const int* s_item, uint32_t& t, double alpha, bool xzero, double* __restrict__ x,
                            double* __restrict__ r, double* part, double (*ired)[32],
                            unsigned long long* pf = nullptr, const TBatchCtx* bc = nullptr) {
    const int NXY = g.NX * g.NY, sy = g.NX, RX = tp.RX;
    constexpr int NT = NCW * 32;
    int cur_sys = -1;
    TRing cur;
    cur.set(tp, t);
    while (true) {
        t_wait_full(full, cur);
        if (pf && threadIdx.x == 0) { *pf = t_ns(); pf = nullptr; }
        int item = s_item[cur.s];
        if (item < 0) { t_release(empty, cur); cur.adv(tp); t = cur.t; return; }
        if (BATCH) {
            const int sy_ = (int)tp.iid.div((uint32_t)item);
            item -= sy_ * tp.I;
            const PcgParams& Q = bc->Ps[sy_];
            if (sy_ != cur_sys) { t_batch_table<NCW>(g, T, Q); cur_sys = sy_; }
            x = Q.T;
            r = Q.r;
            alpha = bc->alpha[sy_];
            part = Q.part + kTPartItems + tp.I;
        }
        const TItem it = t_item(g, tp, item);
        TNodes<NPT, NT> nd;
        nd.init(g, it);
        // stage layout of p: rows j0 - 1 .. j1 (row j0 - 1 of the bottom row block and row
        // j1 of the top one are not loaded; their words stay finite)
        const int jlo = it.j0 - 1;
        double prev[NPT];
        if (it.k0 > 0) {          // halo plane k0 - 1: only the own-node values are needed
            const int kb = (it.k0 - 1) * NXY;
            const int om = cur.s * tp.stage - t_abeg(kb + jlo * g.NX);
#pragma unroll
            for (int m = 0; m < NPT; ++m) prev[m] = (nd.fl[m] & kFOk) ? t_sm[om + kb + nd.off[m]] : 0.0;
            t_release(empty, cur);
            cur.adv(tp);
        } else {
#pragma unroll
            for (int m = 0; m < NPT; ++m) prev[m] = 0.0;
        }
        // Lean planes (2 <= k <= NZ - 2: z class 1, both z neighbours on free planes; x
        // stored): the node's coefficients are item constants in registers, one coupling
        // per neighbour, zero where the neighbour is absent or Dirichlet (its address
        // holds a finite value: another node's, or zeroed ring words); identity rows
        // carry diag = 1 and zero couplings (q = p), threads without a node all zeros.
        double dg[NPT], cxm[NPT], cxp[NPT], cym[NPT], cyp[NPT], c2[NPT], ivd[NPT];
        constexpr bool kLean = NPT <= 2;
        if (kLean) {
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                const int cl = nd.cxy[m] + 9;
                const unsigned f = nd.fl[m];
                const bool ok = f & kFOk;
                const bool cpl = ok && T.nd[cl] != 0.0;
                dg[m] = ok ? T.diag[cl] : 0.0;
                ivd[m] = T.invd[cl];
                cxm[m] = (cpl && (f & kFXm)) ? T.c[0][cl] : 0.0;
                cxp[m] = (cpl && (f & kFXp)) ? T.c[0][cl] : 0.0;
                cym[m] = (cpl && (f & kFYm)) ? T.c[1][cl] : 0.0;
                cyp[m] = (cpl && (f & kFYp)) ? T.c[1][cl] : 0.0;
                c2[m] = (cpl && (f & kFCol)) ? T.c[2][cl] : 0.0;
            }
        }
        uint32_t sm0 = smem_u32(t_sm), sy8 = 8u * (uint32_t)sy, rx8 = 8u * (uint32_t)RX;
        asm volatile("" : "+r"(sm0), "+r"(sy8), "+r"(rx8));
        double acc[2] = {0.0, 0.0};
        for (int k = it.k0; k < it.k1; ++k) {
            const bool nxt = k + 1 < g.NZ;
            const TRing nx = cur.next(tp);
            t_wait_full(full, cur);
            if (nxt) t_wait_full(full, nx);
            const int kb = k * NXY;
            const int oc = cur.s * tp.stage - t_abeg(kb + jlo * g.NX);
            const int op = nxt ? nx.s * tp.stage - t_abeg(kb + NXY + jlo * g.NX) : 0;
            const int ox = cur.s * tp.stage + tp.RB - t_abeg(kb + it.j0 * g.NX);
            if (kLean && !xzero && k >= 2 && k <= g.NZ - 2) {
                const uint32_t b0 = sm0 + 8u * (uint32_t)(oc + kb), b1 = sm0 + 8u * (uint32_t)(op + kb + NXY);
                const uint32_t bx = sm0 + 8u * (uint32_t)(ox + kb);
#pragma unroll
                for (int m = 0; m < NPT; ++m) {
                    const uint32_t o8 = 8u * (uint32_t)nd.off[m];
                    const uint32_t a0 = b0 + o8;
                    const double pp = lds64(a0);
                    const double xm = lds64(a0 - 8u), xp = lds64(a0 + 8u);
                    const double ym = lds64(a0 - sy8), yp = lds64(a0 + sy8);
                    const double zp = lds64(b1 + o8);
                    const double xo = lds64(bx + o8), ro = lds64(bx + rx8 + o8);
                    const double qv = dg[m] * pp - (((cxm[m] * xm + cxp[m] * xp) + (cym[m] * ym + cyp[m] * yp)) +
                                                    c2[m] * (prev[m] + zp));
                    const double xv = __dadd_rn(xo, __dmul_rn(alpha, pp));
                    const bool ok = nd.fl[m] & kFOk;
                    const double rv = ok ? __dsub_rn(ro, __dmul_rn(alpha, qv)) : 0.0;
                    if (ok) {
                        const int p = kb + nd.off[m];
                        x[p] = xv;
                        r[p] = rv;
                    }
                    acc[0] += rv * __dmul_rn(ivd[m], rv);
                    acc[1] += rv * rv;
                    prev[m] = pp;
                }
            } else {
            const int cz9 = 9 * axis_class(k, g.nc[2]);
            const bool zm_ok = k >= 2, zp_ok = nxt;
#pragma unroll
            for (int m = 0; m < NPT; ++m) {
                const unsigned f = nd.fl[m];
                if (!(f & kFOk)) continue;
                const int p = kb + nd.off[m];
                const int cl = nd.cxy[m] + cz9;
                const double pp = t_sm[oc + p];
                double qv;
                if (T.nd[cl] == 0.0) {
                    qv = pp;                              // identity row
                } else {
                    const double xm = (f & kFXm) ? t_sm[oc + p - 1] : 0.0;
                    const double xp = (f & kFXp) ? t_sm[oc + p + 1] : 0.0;
                    const double ym = (f & kFYm) ? t_sm[oc + p - sy] : 0.0;
                    const double yp = (f & kFYp) ? t_sm[oc + p + sy] : 0.0;
                    const double zm = (zm_ok && (f & kFCol)) ? prev[m] : 0.0;
                    const double zp = (zp_ok && (f & kFCol)) ? t_sm[op + p + NXY] : 0.0;
                    qv = T.diag[cl] * pp - ((T.c[0][cl] * (xm + xp) + T.c[1][cl] * (ym + yp)) + T.c[2][cl] * (zm + zp));
                }
                const double iv = T.invd[cl];
                const double xv = __dadd_rn(xzero ? 0.0 : t_sm[ox + p], __dmul_rn(alpha, pp));
                const double rv = __dsub_rn(t_sm[ox + RX + p], __dmul_rn(alpha, qv));
                x[p] = xv;
                r[p] = rv;
                acc[0] += rv * __dmul_rn(iv, rv);
                acc[1] += rv * rv;
                prev[m] = pp;
            }
            }
            t_release(empty, cur);
            cur.adv(tp);
        }
        if (it.k1 < g.NZ) { t_release(empty, cur); cur.adv(tp); }   // the forward halo plane k1
        t_item_sum<2, NCW>(acc, ired, part, tp.I, item);
        t = cur.t;
    }
}

// Fixed-order sum of I item partials per value by the whole CTA (every CTA bitwise equal):
// thread t adds items t, t + B, ... in order (loads batched), then the deterministic
// block_sum.
template <int NV>
__device__ __forceinline__ void t_grid_sum(const double* part, int I, double* red, double* out) {
    const int B = blockDim.x;
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double acc = 0.0;
        int b = threadIdx.x;
        for (; b + 3 * B < I; b += 4 * B) {
            const double v0 = __ldcg(part + k * I + b), v1 = __ldcg(part + k * I + b + B);
            const double v2 = __ldcg(part + k * I + b + 2 * B), v3 = __ldcg(part + k * I + b + 3 * B);
            acc += v0; acc += v1; acc += v2; acc += v3;
        }
        for (; b < I; b += B) acc += __ldcg(part + k * I + b);
        s[k] = acc;
    }
    block_sum<NV>(s, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) out[k] = s[k];
    __syncthreads();
}

// ---- k_t_cg: the CG iterations (cooperative, one CTA per SM, NCW + 1 warps). ----------
// Reads k_s_rhs's Grhs partials; writes the same SolveInfoDev fields as k_s_cg.
template <int NCW, int NPT>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_t_cg(PcgParams P, int Grhs, TPlan tp) {
    cg::grid_group grid = cg::this_grid();
    __shared__ ClassTable T;
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    __shared__ double ired[2][32];
    __shared__ __align__(8) uint64_t full[kTMaxStages], empty[kTMaxStages];
    __shared__ int s_item[kTMaxStages];
    const Grid& g = P.g;
    if (threadIdx.x == 0) {
        for (int s = 0; s < tp.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    build_class_table(T, threadIdx.x, P.mbase, P.cbase, g.dkind);
    t_zero_ring(tp, t_sm);
    {
        const int s[2] = {0, 1};
        grid_sum_wide<2>(P.part, s, Grhs, red, tot);   // also syncs T, the barriers and the ring
    }
    const bool producer = (threadIdx.x >> 5) == NCW;
    const bool plane0 = producer && (threadIdx.x & 31) == 0;
    unsigned* ctr = reinterpret_cast<unsigned*>(P.part + kTCounter);
    double* part = P.part + kTPartItems;
    const double bb = tot[0];
    double rz = tot[1];
    const double bnorm = sqrt(bb);
    const double atol = P.rtol * bnorm;
    double rnorm = bnorm;
    int it = 0, status = 0;
    double rho_prev = 1.0;
    double* pold = P.p0;
    double* pnew = P.p1;
    uint32_t t = 0;          // ring position (identical sequence on producer and consumers)
    unsigned seq = 0;        // sweep sequence number (counter slot seq & 3)
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
            // light RHS: in the first iteration r0 is b and x0 is 0 (neither was written)
            const bool light0 = first && P.light_rhs;
            const double* r0 = light0 ? P.b : P.r;
            unsigned long long* pf = (tp.prof && it == 3) ? tp.prof + 1024 + 16 * blockIdx.x : nullptr;
#define TL_TSTAMP(e) if (pf && threadIdx.x == 0) pf[e] = t_ns();
            TL_TSTAMP(0)
            // ---- sweep A ----
            if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(seq + 2) & 3] = 0u;
            if (producer) {
                if (plane0) t_produce<false>(g, tp, t_sm, full, empty, s_item, ctr + (seq & 3), t, first, r0, pold,
                                             nullptr, nullptr);
            } else {
                t_consume_a<NCW, NPT>(g, tp, T, full, empty, s_item, t, first, beta, pnew, part, ired,
                                      pf ? pf + 1 : nullptr);
                fence_proxy_async_global();
            }
            TL_TSTAMP(2)
            ++seq;
            grid.sync();
            TL_TSTAMP(3)
            t = __shfl_sync(0xffffffffu, t, 0);     // producer warp: lane 0 holds the position
            fence_proxy_async_global();
            t_grid_sum<1>(part, tp.I, red, tot);
            TL_TSTAMP(4)
            const double alpha = rho / tot[0];
            // ---- sweep B ----
            if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(seq + 2) & 3] = 0u;
            if (producer) {
                if (plane0) t_produce<true>(g, tp, t_sm, full, empty, s_item, ctr + (seq & 3), t, false, r0, nullptr,
                                            pnew, light0 ? nullptr : P.T, tp.snake != 0);
            } else {
                // sweep B's item partials go to slots 1, 2: a CTA that is still summing sweep
                // A's slot-0 partials after the barrier must not see them overwritten
                t_consume_b<NCW, NPT>(g, tp, T, full, empty, s_item, t, alpha, light0, P.T, P.r, part + tp.I, ired,
                                      pf ? pf + 5 : nullptr);
                fence_proxy_async_global();
            }
            TL_TSTAMP(6)
            ++seq;
            grid.sync();
            TL_TSTAMP(7)
            t = __shfl_sync(0xffffffffu, t, 0);
            fence_proxy_async_global();
            t_grid_sum<2>(part + tp.I, tp.I, red, tot);
            TL_TSTAMP(8)
#undef TL_TSTAMP
            rz = tot[0];
            rnorm = sqrt(tot[1]);
            rho_prev = rho;
            double* tmp = pold; pold = pnew; pnew = tmp;
            ++it;
        }
    }
    if (it == 0 && P.light_rhs)             // no iteration ran: x0 = 0 was never written
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) P.T[p] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.info->iterations = (status == 1) ? P.maxiter : it;
        P.info->status = status;
        P.info->bnorm = bnorm;
        P.info->rnorm = rnorm;
    }
}

// ---- k_tb_cg: B independent solves on grids of one shape, in lockstep (config 5) ---------
// The scenarios of BASELINE config 5 share the geometry, so the i-th micro solve of all of
// them is ONE launch: the sweeps stream every active system's planes (global item =
// system * I + item), the two grid barriers of an iteration are shared by all systems, and
// each system keeps its own scalars, stop test and iteration count (finished systems drop
// out of the sweeps).  A cfg2-sized solve alone is L2-resident and barrier-bound; 64 of
// them together are an HBM-sized stream (33M nodes) whose barriers amortise over the batch.
// Per-system arithmetic is k_t_cg's: the same item plan gives bitwise the same iterates.
// Per-system sums: warp w adds the partials of systems w, w + nw, ... (lane-strided in a
// fixed order, then the butterfly), every CTA identically.
template <int NV>
__device__ __forceinline__ void tb_sums(const PcgParams* Ps, int B, const int* skip, int off, int stride, int count,
                                        double (*out)[kTBMax]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int s = w; s < B; s += nw) {
        if (skip && skip[s]) continue;
        const double* part = Ps[s].part + off;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double acc = 0.0;
            for (int b = lane; b < count; b += 32) acc += __ldcg(part + v * stride + b);
            acc = warp_sum(acc);
            if (lane == 0) out[v][s] = acc;
        }
    }
    __syncthreads();
}

template <int NCW, int NPT>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_tb_cg(const PcgParams* Ps, int B, int Grhs, TPlan tp,
                                                             unsigned* ctr) {
    cg::grid_group grid = cg::this_grid();
    __shared__ ClassTable T;
    __shared__ __align__(16) unsigned char gbuf[sizeof(Grid)];          // (Grid has default member initialisers)
    Grid& g = *reinterpret_cast<Grid*>(gbuf);
    __shared__ double ired[2][32];
    __shared__ __align__(8) uint64_t full[kTMaxStages], empty[kTMaxStages];
    __shared__ int s_item[kTMaxStages];
    __shared__ double s_alpha[kTBMax], s_beta[kTBMax], s_rho[kTBMax], s_rhop[kTBMax], s_atol[kTBMax];
    __shared__ double s_rnorm[kTBMax], s_bnorm[kTBMax], s_sum[2][kTBMax];
    __shared__ int s_done[kTBMax], s_status[kTBMax], s_its[kTBMax], s_active;
    for (int e = threadIdx.x; e < (int)(sizeof(Grid) / 4); e += blockDim.x)
        reinterpret_cast<uint32_t*>(gbuf)[e] = reinterpret_cast<const uint32_t*>(&Ps[0].g)[e];
    if (threadIdx.x == 0) {
        for (int s = 0; s < tp.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    t_zero_ring(tp, t_sm);
    __syncthreads();
    tb_sums<2>(Ps, B, nullptr, 0, Grhs, Grhs, s_sum);        // b.b and r0.z of every system
    if (threadIdx.x < B) {
        const int s = threadIdx.x;
        const double bb = s_sum[0][s];
        s_bnorm[s] = sqrt(bb);
        s_atol[s] = Ps[s].rtol * s_bnorm[s];
        s_rnorm[s] = s_bnorm[s];
        s_rho[s] = s_sum[1][s];
        s_rhop[s] = 1.0;
        s_done[s] = bb == 0.0 ? 1 : 0;          // b = 0: x = 0 (fem.py:275-276)
        s_status[s] = 0;
        s_its[s] = 0;
    }
    __syncthreads();
    const bool producer = (threadIdx.x >> 5) == NCW;
    const bool plane0 = producer && (threadIdx.x & 31) == 0;
    int it = 0;
    uint32_t t = 0;
    unsigned seq = 0;
    while (true) {
        if (threadIdx.x < B && !s_done[threadIdx.x]) {
            const int s = threadIdx.x;
            int st = -1;
            if (it >= Ps[s].maxiter) st = 1;              // scipy: the limit before the residual
            else if (s_rnorm[s] < s_atol[s]) st = 0;
            else if (!isfinite(s_rnorm[s])) st = 3;
            if (st >= 0) {
                s_done[s] = 1;
                s_status[s] = st;
                s_its[s] = st == 1 ? Ps[s].maxiter : it;
            } else {
                s_beta[s] = it > 0 ? s_rho[s] / s_rhop[s] : 0.0;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int a = 0;
            for (int s = 0; s < B; ++s) a += s_done[s] ? 0 : 1;
            s_active = a;
        }
        __syncthreads();
        if (s_active == 0) break;
        const bool first = it == 0;
        TBatchCtx bc{Ps, s_done, s_alpha, s_beta, B, it & 1, first ? 1 : 0};
        // ---- sweep A ----
        if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(seq + 2) & 3] = 0u;
        if (producer) {
            if (plane0) t_produce<false, true>(g, tp, t_sm, full, empty, s_item, ctr + (seq & 3), t, first, nullptr,
                                               nullptr, nullptr, nullptr, false, &bc);
        } else {
            t_consume_a<NCW, NPT, true>(g, tp, T, full, empty, s_item, t, first, 0.0, nullptr, nullptr, ired, nullptr,
                                        &bc);
            fence_proxy_async_global();
        }
        ++seq;
        grid.sync();
        t = __shfl_sync(0xffffffffu, t, 0);
        fence_proxy_async_global();
        tb_sums<1>(Ps, B, s_done, kTPartItems, tp.I, tp.I, s_sum);
        if (threadIdx.x < B && !s_done[threadIdx.x]) s_alpha[threadIdx.x] = s_rho[threadIdx.x] / s_sum[0][threadIdx.x];
        __syncthreads();
        // ---- sweep B ----
        if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(seq + 2) & 3] = 0u;
        if (producer) {
            if (plane0) t_produce<true, true>(g, tp, t_sm, full, empty, s_item, ctr + (seq & 3), t, false, nullptr,
                                              nullptr, nullptr, nullptr, tp.snake != 0, &bc);
        } else {
            t_consume_b<NCW, NPT, true>(g, tp, T, full, empty, s_item, t, 0.0, first, nullptr, nullptr, nullptr, ired,
                                        nullptr, &bc);
            fence_proxy_async_global();
        }
        ++seq;
        grid.sync();
        t = __shfl_sync(0xffffffffu, t, 0);
        fence_proxy_async_global();
        tb_sums<2>(Ps, B, s_done, kTPartItems + tp.I, tp.I, tp.I, s_sum);
        if (threadIdx.x < B && !s_done[threadIdx.x]) {
            const int s = threadIdx.x;
            s_rhop[s] = s_rho[s];
            s_rho[s] = s_sum[0][s];
            s_rnorm[s] = sqrt(s_sum[1][s]);
        }
        __syncthreads();
        ++it;
    }
    // systems that ran no iteration (b = 0): x0 = 0 was never written (light RHS)
    for (int s = 0; s < B; ++s)
        if (s_its[s] == 0 && s_status[s] != 1)
            for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) Ps[s].T[p] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x < B) {
        const int s = threadIdx.x;
        SolveInfoDev* info = Ps[s].info;
        info->iterations = s_its[s];
        info->status = s_status[s];
        info->bnorm = s_bnorm[s];
        info->rnorm = s_rnorm[s];
    }
}

}  // namespace tl
