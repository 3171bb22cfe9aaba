// tl_2d.cuh — the 2D (P1 triangle / 5-point) variants of the step kernels (SURVEY §8f
// row 4), sm_100a, fp64.
//
// The reference's 2D meshes (lpbfsim/mesh.py:84-93,388-439) split every cell of the
// structured grid into the triangles [0,1,3] and [0,3,2] (corner = dx + 2 dy), both
// positively oriented:
//     tri 0: (0,0) (1,0) (1,1)        tri 1: (0,0) (1,1) (0,1)
// Right triangles with axis-aligned legs: the P1 gradients are axis-aligned, the element
// stiffness kbar area grad_i.grad_j (fem.py:170) couples only the leg endpoints
// (-kbar area / h_a^2 on the leg along axis a) and the hypotenuse carries nothing, so with
// the row-sum lumped mass (fem.py:167-169) the assembled operator is the 5-point stencil
//     (A x)_p = diag_p x_p - sum_{a in x,y} (w_a[p] x_{p+e_a} + w_a[p-e_a] x_{p-e_a}).
// A 2D grid is a tl::Grid with nc[2] = 0 (NZ = 1): the constrained system, the Jacobi-PCG
// (k_vc_cg), the increment and lag kernels of tl_vc.cuh run unchanged on it (their z
// terms are guarded by 0 < k < nc[2]); only the assembly, the interpolation and the mass
// norms have triangle variants here.  Element quadrature: the three edge midpoints,
// weights 1/3 (mesh.py:107-110); boundary edges: two Gauss points (mesh.py:129-131).  The
// vertical axis is y: BOTTOM / TOP are y = lo / y = hi (mesh.py:206-209), so the Robin
// terms (fem.py:241-268) sit on the top row j = nc[1].  Beam: gaussian_source_2d
// (sources.py:57-64), peak = P eta / (r d) passed in Gauss::peak.
// oracle/tri2d.py restates the same arrays in numpy (checked against the reference's CSR
// matrix and RHS to 3e-15).
#pragma once

#include "tl_vc.cuh"

namespace tl {

__host__ __device__ __forceinline__ bool grid_is_2d(const Grid& g) { return g.nc[2] == 0; }

// vertex offsets (dx, dy) of the two triangles, in the reference's vertex order
__constant__ int8_t c_tri[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {1, 1}, {0, 1}}};
// legs of each triangle: (lower vertex, upper vertex, axis)
__constant__ int8_t c_leg[2][2][3] = {{{0, 1, 0}, {1, 2, 1}}, {{0, 2, 1}, {2, 1, 0}}};
// barycentric quadrature points (rows) of the triangle rule
__constant__ double c_qphi2[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};

// Phase 1, one thread per (cell, triangle): kbar, the lumped mass of each vertex (times
// area) and the Gaussian load of each vertex (times area); slots of 4 per element as in 3D.
__global__ void k_vc_tris(Grid g, VcMat Mi, VcMat Mo, VcRegion R, const double* __restrict__ T_old,
                          const double* __restrict__ T_lag, double dt, Gauss src, double* __restrict__ tk,
                          double* __restrict__ tml, double* __restrict__ tsrc) {
    const double area = 0.5 * g.h[0] * g.h[1];
    const int ncell = g.nc[0] * g.nc[1];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * ncell; e += gridDim.x * blockDim.x) {
        const int c = e >> 1, t = e & 1;
        const int cell[2] = {c % g.nc[0], c / g.nc[0]};
        double Tl[3], To[3];
        for (int v = 0; v < 3; ++v) {
            const int id = (cell[0] + c_tri[t][v][0]) + g.NX * (cell[1] + c_tri[t][v][1]);
            Tl[v] = T_lag[id];
            To[v] = T_old[id];
        }
        bool inside = true;
        if (R.piecewise || R.latent_inside) {
            for (int a = 0; a < 2; ++a) {
                double sx = 0.0;
                for (int v = 0; v < 3; ++v) sx += node_coord(g, a, cell[a] + c_tri[t][v][a]);
                const double cen = sx / 3.0;
                inside = inside && cen >= R.lo[a] && cen <= R.hi[a];
            }
        }
        const VcMat& M = (R.piecewise && !inside) ? Mo : Mi;
        const bool lat_on = M.latent && (!R.latent_inside || inside);
        const double w3 = 1.0 / 3.0;
        double kbar = 0.0, ml[3] = {0.0, 0.0, 0.0}, qs[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < 3; ++q) {
            double tq = 0.0, tqo = 0.0;
            for (int v = 0; v < 3; ++v) {
                tq += c_qphi2[q][v] * Tl[v];
                tqo += c_qphi2[q][v] * To[v];
            }
            const double kq = vc_interp(tq, M.kT, M.kv, M.nk);
            double cq = vc_interp(tq, M.cT, M.cv, M.nc);
            if (lat_on) cq += vc_latent(M, tq, tqo);
            kbar += w3 * kq;
            const double mq = w3 * (M.rho * cq / dt);
            double Qq = 0.0;
            if (src.on) {
                double x[2];
                for (int a = 0; a < 2; ++a) {
                    double sx = 0.0;
                    for (int v = 0; v < 3; ++v) sx += c_qphi2[q][v] * node_coord(g, a, cell[a] + c_tri[t][v][a]);
                    x[a] = sx;
                }
                const double ux = (x[0] - src.center[0]) / src.radius, uy = (x[1] - src.center[1]) / src.depth;
                Qq = w3 * (src.peak * exp(-(ux * ux + uy * uy)));
            }
            for (int r = 0; r < 3; ++r) {
                ml[r] += mq * c_qphi2[q][r];
                qs[r] += Qq * c_qphi2[q][r];
            }
        }
        tk[e] = kbar;
        for (int r = 0; r < 3; ++r) {
            tml[4 * (size_t)e + r] = ml[r] * area;
            tsrc[4 * (size_t)e + r] = qs[r] * area;
        }
    }
}

// Phase 2, one thread per node: gather the (up to six) triangles touching the node in a
// fixed order (no atomics), then the lumped Robin terms of the adjacent top edges.
__global__ void k_vc_assemble2(Grid g, const double* __restrict__ tk, const double* __restrict__ tml,
                               const double* __restrict__ tsrc, const double* __restrict__ T_old,
                               const double* __restrict__ T_lag, const double* __restrict__ extra, VcRobin rb,
                               double* __restrict__ diag, double* __restrict__ wx, double* __restrict__ wy,
                               double* __restrict__ wz, double* __restrict__ b) {
    const double area = 0.5 * g.h[0] * g.h[1];
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
        const int i = p % g.NX, j = p / g.NX;
        const double Top = T_old[p];
        double dg = 0.0, bb = 0.0, wf[2] = {0.0, 0.0};
        for (int o = 0; o < 4; ++o) {
            const int oi = o & 1, oj = o >> 1;
            const int ci = i - oi, cj = j - oj;
            if (ci < 0 || cj < 0 || ci >= g.nc[0] || cj >= g.nc[1]) continue;
            const int c = ci + g.nc[0] * cj;
            for (int t = 0; t < 2; ++t) {
                int r = -1;
                for (int v = 0; v < 3; ++v)
                    if (c_tri[t][v][0] == oi && c_tri[t][v][1] == oj) r = v;
                if (r < 0) continue;
                const size_t e = 2 * (size_t)c + t;
                const double ml = tml[4 * e + r];
                const double kbar = tk[e];
                dg += ml;
                bb += ml * Top + tsrc[4 * e + r];
                for (int l = 0; l < 2; ++l) {
                    const int va = c_leg[t][l][0], vb = c_leg[t][l][1], ax = c_leg[t][l][2];
                    if (r != va && r != vb) continue;
                    const double we = kbar * area / (g.h[ax] * g.h[ax]);
                    dg += we;
                    if (r == va) wf[ax] += we;      // the leg's lower node holds its weight
                }
            }
        }
        if (rb.on && j == g.nc[1]) {
            // top edges [il, il + 1]; facet nodes in the reference's order (right, left):
            // the facet of [n00, n11, n01] that omits vertex 0 (mesh.py:190-192)
            const double g2 = 0.5 / sqrt(3.0);
            const double fphi[2][2] = {{0.5 + g2, 0.5 - g2}, {0.5 - g2, 0.5 + g2}};
            const double load = rb.h * rb.Tamb + rb.se * (rb.Tamb * rb.Tamb * rb.Tamb * rb.Tamb);
            for (int il = i - 1; il <= i; ++il) {
                if (il < 0 || il >= g.nc[0]) continue;
                const double Tr = T_lag[(il + 1) + g.NX * j], Tleft = T_lag[il + g.NX * j];
                const int me = (il + 1 == i) ? 0 : 1;
                for (int q = 0; q < 2; ++q) {
                    const double tq = fphi[q][0] * Tr + fphi[q][1] * Tleft;
                    const double coeff = rb.h + rb.se * (tq * tq * tq);
                    dg += 0.5 * coeff * fphi[q][me] * g.h[0];
                    bb += 0.5 * load * fphi[q][me] * g.h[0];
                }
            }
        }
        if (extra) bb += extra[p];
        diag[p] = dg;
        wx[p] = wf[0];
        wy[p] = wf[1];
        wz[p] = 0.0;
        b[p] = bb;
    }
}

// P1 interpolant of v on the triangle lattice at (x, y) (Mesh.locate / interpolate,
// mesh.py:308-361): cell by floor (clipped), triangle 0 where xi >= eta (the first
// candidate wins ties; on the diagonal both give the same value), P1 inside it.
__device__ __forceinline__ double p1_eval2(const Grid& G, const double* v, double x, double y) {
    const double pt[2] = {x, y};
    int c[2];
    double xi[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        int ci = (int)floor((pt[a] - (G.lo0[a] + G.off[a])) / G.h[a]);
        ci = ci < 0 ? 0 : (ci > G.nc[a] - 1 ? G.nc[a] - 1 : ci);
        c[a] = ci;
        xi[a] = (pt[a] - node_coord(G, a, ci)) / G.h[a];
    }
    const int p0 = c[0] + G.NX * c[1];
    const double v00 = v[p0], v11 = v[p0 + G.NX + 1];
    if (xi[0] >= xi[1]) return (1.0 - xi[0]) * v00 + (xi[0] - xi[1]) * v[p0 + 1] + xi[1] * v11;
    return (1.0 - xi[1]) * v00 + xi[0] * v11 + (xi[1] - xi[0]) * v[p0 + G.NX];
}

// Global field at the nodes of a 2D local lattice (trace, relocation, error metrics);
// gamma_only: lateral (i = 0, NX-1) and bottom (j = 0) nodes only, the others untouched.
__global__ void k_interp2(Grid G, Grid L, const double* __restrict__ vg, double* __restrict__ out, int gamma_only) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L.n; p += gridDim.x * blockDim.x) {
        const int i = p % L.NX, j = p / L.NX;
        if (gamma_only && !(i == 0 || i == L.nc[0] || j == 0)) continue;
        out[p] = p1_eval2(G, vg, node_coord(L, 0, i), node_coord(L, 1, j));
    }
}

__global__ void k_interp_nodes2(Grid G, Grid L, const double* __restrict__ vg, const int* __restrict__ idx, int n,
                                double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int p = idx[e];
        if (p < 0 || p >= L.n) { out[e] = nan(""); continue; }
        out[e] = p1_eval2(G, vg, node_coord(L, 0, p % L.NX), node_coord(L, 1, p / L.NX));
    }
}

__global__ void k_interp_pts2(Grid G, const double* __restrict__ vg, const double* __restrict__ pts, int npts,
                              double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < npts; e += gridDim.x * blockDim.x)
        out[e] = p1_eval2(G, vg, pts[2 * e], pts[2 * e + 1]);
}

// v^T M v with the consistent P1 mass matrix of the triangles (fem.mass_matrix,
// fem.py:434-446): per triangle area/12 (sum v_i^2 + (sum v_i)^2); d = a - b (d = a when
// b == nullptr) -> part[2 blk], b -> part[2 blk + 1].
__global__ void k_mass_norms2(Grid L, const double* __restrict__ a, const double* __restrict__ b, double* part) {
    __shared__ double red[64];
    const int ncell = L.nc[0] * L.nc[1];
    double acc[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const int p0 = (c % L.nc[0]) + L.NX * (c / L.nc[0]);
        const int off[4] = {0, 1, L.NX, L.NX + 1};
        double d[4], r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double av = a[p0 + off[q]];
            const double bv = b ? b[p0 + off[q]] : 0.0;
            d[q] = b ? av - bv : av;
            r[q] = bv;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int m = t == 0 ? 1 : 2;          // (0,0) m (1,1): the triangle's third corner
            const double s1 = d[0] + d[m] + d[3];
            acc[0] += d[0] * d[0] + d[m] * d[m] + d[3] * d[3] + s1 * s1;
            const double s2 = r[0] + r[m] + r[3];
            acc[1] += r[0] * r[0] + r[m] * r[m] + r[3] * r[3] + s2 * s2;
        }
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        const double w = 0.5 * L.h[0] * L.h[1] / 12.0;
        part[2 * blockIdx.x] = acc[0] * w;
        part[2 * blockIdx.x + 1] = acc[1] * w;
    }
}

// Masked mass norms in 2D (twolevel.masked_mass, twolevel.py:361-373): (a-b)^T M (a-b) over
// the triangles whose centroid lies in the closed box -> part[2 blk], the others ->
// part[2 blk + 1]; per triangle area/12 (sum d_i^2 + (sum d_i)^2) as k_mass_norms2.
__global__ void k_mass_norms_split2(Grid L, const double* __restrict__ a, const double* __restrict__ b,
                                    double blo0, double blo1, double bhi0, double bhi1, double* part) {
    __shared__ double red[64];
    const int ncell = L.nc[0] * L.nc[1];
    const double blo[2] = {blo0, blo1}, bhi[2] = {bhi0, bhi1};
    double acc[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const int cell[2] = {c % L.nc[0], c / L.nc[0]};
        for (int t = 0; t < 2; ++t) {
            double d[3];
            bool in = true;
            for (int v = 0; v < 3; ++v) {
                const int id = (cell[0] + c_tri[t][v][0]) + L.NX * (cell[1] + c_tri[t][v][1]);
                d[v] = a[id] - b[id];
            }
            for (int ax = 0; ax < 2; ++ax) {
                double sx = 0.0;
                for (int v = 0; v < 3; ++v) sx += node_coord(L, ax, cell[ax] + c_tri[t][v][ax]);
                const double cen = sx / 3.0;
                in = in && cen >= blo[ax] && cen <= bhi[ax];
            }
            const double s1 = d[0] + d[1] + d[2];
            acc[in ? 0 : 1] += d[0] * d[0] + d[1] * d[1] + d[2] * d[2] + s1 * s1;
        }
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        const double w = 0.5 * L.h[0] * L.h[1] / 12.0;
        part[2 * blockIdx.x] = acc[0] * w;
        part[2 * blockIdx.x + 1] = acc[1] * w;
    }
}

// Full-mode overlap feedback in 2D (twolevel._overlap_feedback, twolevel.py:186-239; the 3D
// kernel is k_overlap_feedback in tl_vc.cuh): per global node, over the (up to six) global
// triangles touching it and their three edge-midpoint quadrature points that lie in the
// closed local box, the local fields are located in the local lattice (cell by floor,
// triangle 0 where xi >= eta, as p1_eval2) and the density
//   -(c_eff,l rho_l k_g/k_l - c_g rho_g) dT/dt + ((k_g/k_l) k_l' - k_g') |grad T|^2 + (k_g/k_l - 1) Q
// is gathered as w_q area density phi_i(x_q) (no atomics).
__global__ void k_overlap_feedback2(Grid G, Grid L, const double* __restrict__ Tn, const double* __restrict__ To,
                                    double dt, VcMat Mg, VcMat Ml, Gauss src, double* __restrict__ load) {
    const double area = 0.5 * G.h[0] * G.h[1];
    double llo[2], lhi[2];
    for (int a = 0; a < 2; ++a) {
        llo[a] = node_coord(L, a, 0);
        lhi[a] = node_coord(L, a, L.nc[a]);
    }
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < G.n; p += gridDim.x * blockDim.x) {
        const int idx[2] = {p % G.NX, p / G.NX};
        double acc = 0.0;
        for (int o = 0; o < 4; ++o) {
            const int oo[2] = {o & 1, (o >> 1) & 1};
            const int cell[2] = {idx[0] - oo[0], idx[1] - oo[1]};
            if (cell[0] < 0 || cell[0] >= G.nc[0] || cell[1] < 0 || cell[1] >= G.nc[1]) continue;
            for (int t = 0; t < 2; ++t) {
                int r = -1;
                for (int v = 0; v < 3; ++v)
                    if (c_tri[t][v][0] == oo[0] && c_tri[t][v][1] == oo[1]) r = v;
                if (r < 0) continue;
                for (int q = 0; q < 3; ++q) {
                    if (c_qphi2[q][r] == 0.0) continue;          // the point on the opposite edge
                    double x[2];
                    bool in = true;
                    for (int a = 0; a < 2; ++a) {
                        double sx = 0.0;
                        for (int v = 0; v < 3; ++v) sx += c_qphi2[q][v] * node_coord(G, a, cell[a] + c_tri[t][v][a]);
                        x[a] = sx;
                        in = in && x[a] >= llo[a] && x[a] <= lhi[a];
                    }
                    if (!in) continue;
                    int c[2];
                    double xi[2];
                    for (int a = 0; a < 2; ++a) {
                        int ci = (int)floor((x[a] - (L.lo0[a] + L.off[a])) / L.h[a]);
                        ci = ci < 0 ? 0 : (ci > L.nc[a] - 1 ? L.nc[a] - 1 : ci);
                        c[a] = ci;
                        xi[a] = (x[a] - node_coord(L, a, ci)) / L.h[a];
                    }
                    const int n0 = c[0] + L.NX * c[1], n3 = n0 + L.NX + 1;
                    double Tq, Tqo, gx, gy;
                    if (xi[0] >= xi[1]) {                           // triangle (0,0) (1,0) (1,1)
                        const int n1 = n0 + 1;
                        const double w0 = 1.0 - xi[0], w1 = xi[0] - xi[1], w2 = xi[1];
                        Tq = w0 * Tn[n0] + w1 * Tn[n1] + w2 * Tn[n3];
                        Tqo = w0 * To[n0] + w1 * To[n1] + w2 * To[n3];
                        gx = (Tn[n1] - Tn[n0]) / L.h[0];
                        gy = (Tn[n3] - Tn[n1]) / L.h[1];
                    } else {                                        // triangle (0,0) (1,1) (0,1)
                        const int n2 = n0 + L.NX;
                        const double w0 = 1.0 - xi[1], w1 = xi[0], w2 = xi[1] - xi[0];
                        Tq = w0 * Tn[n0] + w1 * Tn[n3] + w2 * Tn[n2];
                        Tqo = w0 * To[n0] + w1 * To[n3] + w2 * To[n2];
                        gx = (Tn[n3] - Tn[n2]) / L.h[0];
                        gy = (Tn[n2] - Tn[n0]) / L.h[1];
                    }
                    const double gsq = gx * gx + gy * gy;
                    const double kg = tab_interp(Tq, Mg.kT, Mg.kv, Mg.nk);
                    const double kl = tab_interp(Tq, Ml.kT, Ml.kv, Ml.nk);
                    const double ratio = kg / kl;
                    const double ceff = tab_interp(Tq, Ml.cT, Ml.cv, Ml.nc) + Ml.chi * vc_phase_deriv(Ml, Tq);
                    const double cg = tab_interp(Tq, Mg.cT, Mg.cv, Mg.nc);
                    double dens = -(ceff * Ml.rho * ratio - cg * Mg.rho) * ((Tq - Tqo) / dt);
                    dens += (ratio * vc_dkdT(Tq, Ml.kT, Ml.kv, Ml.nk) - vc_dkdT(Tq, Mg.kT, Mg.kv, Mg.nk)) * gsq;
                    if (src.on) {
                        const double ux = (x[0] - src.center[0]) / src.radius, uy = (x[1] - src.center[1]) / src.depth;
                        dens += (ratio - 1.0) * (src.peak * exp(-(ux * ux + uy * uy)));
                    }
                    acc += (1.0 / 3.0) * area * dens * c_qphi2[q][r];
                }
            }
        }
        load[p] = acc;
    }
}

// Interface functional in 2D (twolevel.transmission_load, twolevel.py:159-183; the 3D kernel
// is k_trans_entries): the interface edges of the local lattice are the bottom row
// (nc[0] edges, owner triangle 0 of the cell above, normal -e_y) and the two lateral columns
// (nc[1] edges each; left: owner triangle 1, normal -e_x; right: owner triangle 0, normal
// +e_x) (mesh.py:477-523).  Each edge carries two Gauss points of weight length / 2
// (mesh.py:129-131); dT/dn is the owner triangle's one-sided P1 gradient; jump as in 3D.
// Entry e = 2 f + q writes 3 (global node, density * barycentric) pairs at 3 e + r.
__global__ void k_trans_entries2(Grid G, Grid L, const double* __restrict__ T, double jump, KTab kg, KTab kl,
                                 int nedge, int* __restrict__ keys, int* __restrict__ idx,
                                 double* __restrict__ vals) {
    const double gq = 0.5 / sqrt(3.0);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * nedge; e += gridDim.x * blockDim.x) {
        int f = e >> 1;
        const int q = e & 1;
        int na, nb;                      // the edge's end nodes (local ids)
        double dTdn, len;
        if (f < L.nc[0]) {               // bottom edge of cell (f, 0)
            na = f;
            nb = f + 1;
            dTdn = -(T[nb + L.NX] - T[nb]) / L.h[1];            // triangle 0: gy = (T11 - T10) / hy
            len = L.h[0];
        } else if ((f -= L.nc[0]) < L.nc[1]) {                   // left edge of cell (0, f)
            na = L.NX * f;
            nb = na + L.NX;
            dTdn = -(T[nb + 1] - T[nb]) / L.h[0];               // triangle 1: gx = (T11 - T01) / hx
            len = L.h[1];
        } else {                                                 // right edge of cell (nc0 - 1, f)
            f -= L.nc[1];
            na = L.NX * f + L.nc[0];
            nb = na + L.NX;
            dTdn = (T[na] - T[na - 1]) / L.h[0];                // triangle 0: gx = (T10 - T00) / hx
            len = L.h[1];
        }
        const double wa = q == 0 ? 0.5 + gq : 0.5 - gq, wb = 1.0 - wa;
        const double x = wa * node_coord(L, 0, na % L.NX) + wb * node_coord(L, 0, nb % L.NX);
        const double y = wa * node_coord(L, 1, na / L.NX) + wb * node_coord(L, 1, nb / L.NX);
        double jq = jump;
        if (kg.n > 0) {
            const double tq = wa * T[na] + wb * T[nb];
            jq = tab_interp(tq, kg.T, kg.v, kg.n) - tab_interp(tq, kl.T, kl.v, kl.n);
        }
        const double dens = 0.5 * len * jq * dTdn;
        // locate in the global lattice as p1_eval2 does
        const double pt[2] = {x, y};
        int c[2];
        double xi[2];
        for (int a = 0; a < 2; ++a) {
            int ci = (int)floor((pt[a] - (G.lo0[a] + G.off[a])) / G.h[a]);
            ci = ci < 0 ? 0 : (ci > G.nc[a] - 1 ? G.nc[a] - 1 : ci);
            c[a] = ci;
            xi[a] = (pt[a] - node_coord(G, a, ci)) / G.h[a];
        }
        const int p0 = c[0] + G.NX * c[1];
        int nd[3];
        double w[3];
        nd[0] = p0;
        nd[1] = p0 + G.NX + 1;
        if (xi[0] >= xi[1]) { nd[2] = p0 + 1; w[0] = 1.0 - xi[0]; w[1] = xi[1]; w[2] = xi[0] - xi[1]; }
        else { nd[2] = p0 + G.NX; w[0] = 1.0 - xi[1]; w[1] = xi[0]; w[2] = xi[1] - xi[0]; }
        for (int r = 0; r < 3; ++r) {
            keys[3 * e + r] = nd[r];
            idx[3 * e + r] = 3 * e + r;
            vals[3 * e + r] = dens * w[r];
        }
    }
}

}  // namespace tl
