// tl_grid.cuh — structured Kuhn-P1 grid math shared by all kernels (sm_100a, fp64).
//
// The reference assembles P1 elements on Kuhn-subdivided hexes
// (lpbfsim/mesh.py:84-102,388-439) with a row-sum lumped mass
// (lpbfsim/fem.py:167-169).  For a constant material this is exactly a
// 7-point operator whose weights depend only on how many Kuhn tets touch a
// node / an axis edge (pinned by
// tests/test_oracle_golden.py).  Those counts depend only on whether each
// index sits on the low face, the interior or the high face of its axis, so
// each node falls in one of 3x3x3 = 27 classes; all coefficients are a
// per-class table held in shared memory, rebuilt per solve (dt changes the
// mass term).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tl {

constexpr int kGamma = 1;     // TL_DIRICHLET_GAMMA
constexpr int kBottom = 0;    // TL_DIRICHLET_BOTTOM

// Unsigned division by a run-time invariant (valid for n < 2^31).
struct FastDiv {
    uint32_t d = 1, mul = 0, shr = 0;
    __host__ void init(uint32_t dd) {
        d = dd;
        if (d == 1) { mul = 0; shr = 0; return; }
        uint32_t l = 0;
        while ((1u << l) < d) ++l;
        uint32_t p = 31 + l;
        mul = (uint32_t)(((1ull << p) + d - 1) / d);
        shr = p - 32;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return d == 1 ? n : (__umulhi(n, mul) >> shr);
    }
};

// Device view of one structured grid.
struct Grid {
    int nc[3];          // cells per axis
    int NX, NY, NZ;     // nodes per axis
    int n;              // nodes
    FastDiv divX, divY; // decode id -> (i, j, k)
    double lo0[3], hi0[3], step[3], off[3];   // node coordinates
    double h[3];        // spacing (box.lengths / ncells)
    int dkind;          // Dirichlet set
};

__device__ __forceinline__ void decode(const Grid& g, int p, int& i, int& j, int& k) {
    uint32_t t = g.divX.div((uint32_t)p);
    i = p - (int)t * g.NX;
    uint32_t kk = g.divY.div(t);
    k = (int)kk;
    j = (int)t - k * g.NY;
}

// Axis class: 0 = low face (idx 0), 1 = interior, 2 = high face (idx n).
__device__ __forceinline__ int axis_class(int idx, int ncell) {
    return idx == 0 ? 0 : (idx == ncell ? 2 : 1);
}

// Node coordinate along axis a: numpy.linspace(lo0, hi0, n+1)[idx] + offset,
// with the same two roundings numpy performs (idx*step + start; last = stop).
__device__ __forceinline__ double node_coord(const Grid& g, int a, int idx) {
    double base = (idx == g.nc[a]) ? g.hi0[a] : __dadd_rn(__dmul_rn((double)idx, g.step[a]), g.lo0[a]);
    return __dadd_rn(base, g.off[a]);
}

// Per-class coefficient table (27 classes, class id = cx + 3*cy + 9*cz).
struct ClassTable {
    double diag[27];     // diagonal of A (mass + stiffness)
    double invd[27];     // Jacobi: 1/diag on free rows, 1 on Dirichlet rows
    double mass[27];     // lumped mass (rho c / dt) V n_p / 24
    double c[3][27];     // axis-edge coupling kappa V / h_a^2 * n_e / 6
    double nd[27];       // 1 if the class is a free (non-Dirichlet) node
};

// Incidence counts from the axis classes.
__host__ __device__ inline void class_counts(int cls, int& n_p, int n_e[3], int cnt[3],
                                             int h0[3], int h1[3]) {
    int cl[3] = {cls % 3, (cls / 3) % 3, cls / 9};
    for (int a = 0; a < 3; ++a) {
        h0[a] = cl[a] != 2;   // cell idx exists along a
        h1[a] = cl[a] != 0;   // cell idx-1 exists along a
        cnt[a] = h0[a] + h1[a];
    }
    n_p = 2 * cnt[0] * cnt[1] * cnt[2] + 4 * (h0[0] & h0[1] & h0[2]) + 4 * (h1[0] & h1[1] & h1[2]);
    for (int a = 0; a < 3; ++a) {
        int b = (a + 1) % 3, c = (a + 2) % 3;
        n_e[a] = cnt[b] * cnt[c] + (h0[b] & h0[c]) + (h1[b] & h1[c]);
    }
}

__device__ __forceinline__ bool class_is_dirichlet(int cls, int dkind) {
    int cx = cls % 3, cy = (cls / 3) % 3, cz = cls / 9;
    if (cz == 0) return true;
    if (dkind == kGamma) return cx != 1 || cy != 1;
    return false;
}

// Built by threads [0, 27) of a block; caller syncs.
__device__ inline void build_class_table(ClassTable& T, int t, double mbase, const double cbase[3],
                                         int dkind) {
    if (t >= 27) return;
    int n_p, n_e[3], cnt[3], h0[3], h1[3];
    class_counts(t, n_p, n_e, cnt, h0, h1);
    double m = mbase * (double)n_p;
    double d = m;
    for (int a = 0; a < 3; ++a) {
        double c = cbase[a] * (double)n_e[a];
        T.c[a][t] = c;
        d += c * (double)cnt[a];
    }
    bool D = class_is_dirichlet(t, dkind);
    T.mass[t] = m;
    T.diag[t] = D ? 1.0 : d;
    T.invd[t] = D ? 1.0 : 1.0 / d;    // fem.py:283-284 (diag > 0 always here)
    T.nd[t] = D ? 0.0 : 1.0;
}

}  // namespace tl
