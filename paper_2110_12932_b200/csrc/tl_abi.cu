// tl_abi.cu — C ABI (include/tlgpu.h) over the sm_100a kernels in tl_kernels.cuh.
//
// Host orchestration of one two-level run.  Per macro step of the one-way
// multirate cycle (lpbfsim/multirate.py:105-164, one-way branch :144-155):
//   k_deposit            swept-track deposit for [t, t + dt_macro]       (runner.py:75-79)
//   k_pcg<false>         global backward-Euler step, bottom Dirichlet    (twolevel.py:242-271)
//   k_interp (gamma)     trace_pred = P1(global) on the gamma nodes      (multirate.py:129)
//   m x k_pcg<true>      micro local steps, blended trace, Gaussian      (multirate.py:133-142)
//   [k_pcg<true>]        corrector re-solve of the last interval         (multirate.py:149-150)
//   k_interp (all)       relocation: local = P1(global) at moved nodes  (scanpath.py:243-248)
// All state stays on the device; the host only enqueues launches.
#include <cub/cub.cuh>
#include <algorithm>
#include <initializer_list>
#include <map>
#include <atomic>
#include <mutex>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tlgpu.h"
#include "tl_resident_cg.cuh"
#include "tl_stream.cuh"
#include "tl_tiled.cuh"
#include "tl_slab.cuh"
#include "tl_slabdev.cuh"
#include "tl_vc.cuh"
#include "tl_2d.cuh"

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device, per-function attribute:
// remember the largest size set for each (device, kernel) and raise it when needed.
static cudaError_t ensure_smem_attr(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = set[{dev, fn}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define TL_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(TL_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// Field arguments of the *_host entry points may be host OR device pointers: unified virtual
// addressing tells them apart, so a caller that keeps its fields on the device between calls
// (DeviceVector in paper_2110_12932_b200/_native.py; tl_dev_alloc) pays no PCIe traffic for
// them.  g_h2d_bytes / g_d2h_bytes count what did cross (tl_host_traffic).
std::atomic<long long> g_h2d_bytes{0}, g_d2h_bytes{0};

bool on_device(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// st == nullptr: the legacy default stream, synchronous for host memory
cudaError_t copy_in(void* dst, const void* src, size_t bytes, cudaStream_t st = nullptr, bool async = false) {
    if (!on_device(src)) g_h2d_bytes += (long long)bytes;
    return async ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st) : cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
}

// a device destination is complete when this returns (device-to-device copies are
// asynchronous to the host; the next call may run on another stream)
cudaError_t copy_out(void* dst, const void* src, size_t bytes) {
    const bool dev = on_device(dst);
    if (!dev) g_d2h_bytes += (long long)bytes;
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
    if (e == cudaSuccess && dev) e = cudaStreamSynchronize(nullptr);
    return e;
}

// allow2d: a descriptor with ncells[2] == 0 is a 2D grid (NZ = 1; csrc/tl_2d.cuh); only the
// entry points with triangle variants accept it.
int make_grid(const tl_grid_desc& d, int dkind, tl::Grid& g, bool allow2d = false) {
    const int dim = (allow2d && d.ncells[2] == 0) ? 2 : 3;
    if (dim == 2) {
        g.nc[2] = 0;
        g.lo0[2] = g.hi0[2] = g.off[2] = g.step[2] = 0.0;
        g.h[2] = 1.0;
    }
    for (int a = 0; a < dim; ++a) {
        if (d.ncells[a] < 1) return fail(TL_E_INVALID, "grid needs at least one cell per axis");
        if (!(d.hi0[a] > d.lo0[a])) return fail(TL_E_INVALID, "degenerate grid box");
        g.nc[a] = d.ncells[a];
        g.lo0[a] = d.lo0[a];
        g.hi0[a] = d.hi0[a];
        g.off[a] = d.offset[a];
        g.step[a] = (d.hi0[a] - d.lo0[a]) / (double)d.ncells[a];  // linspace step = delta / div
        g.h[a] = g.step[a];                                         // Box.lengths / ncells
    }
    g.NX = g.nc[0] + 1;
    g.NY = g.nc[1] + 1;
    g.NZ = g.nc[2] + 1;
    long long n = (long long)g.NX * g.NY * g.NZ;
    if (n >= (1ll << 31)) return fail(TL_E_INVALID, "grid exceeds 2^31 nodes");
    g.n = (int)n;
    g.divX.init((uint32_t)g.NX);
    g.divY.init((uint32_t)g.NY);
    g.dkind = dkind;
    return TL_OK;
}

int coop_blocks(bool gauss, size_t smem, int sms, int& blocks) {
    static thread_local int cached[2] = {0, 0};
    static thread_local size_t cached_smem[2] = {0, 0};
    if (cached[gauss] > 0 && cached_smem[gauss] == smem) { blocks = cached[gauss] * sms; return TL_OK; }
    int per_sm = 0;
    cudaError_t e;
    if (gauss)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tl::k_pcg<true>, tl::kTPB, smem);
    else
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tl::k_pcg<false>, tl::kTPB, smem);
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("occupancy: ") + cudaGetErrorString(e));
    if (per_sm < 1) return fail(TL_E_CUDA, "k_pcg cannot be resident");
    cached[gauss] = per_sm;
    cached_smem[gauss] = smem;
    blocks = per_sm * sms;
    return TL_OK;
}

size_t gauss_smem(const tl::Grid& g) { return sizeof(double) * (size_t)tl::gauss_smem_len(g); }

int launch_pcg(tl::PcgParams& P, bool gauss, int sms, cudaStream_t st, int64_t* launches) {
    size_t smem = gauss ? gauss_smem(P.g) : 0;
    if (gauss && smem > 200 * 1024) return fail(TL_E_INVALID, "local grid too long for Gaussian tables");
    int blocks = 0;
    int rc = coop_blocks(gauss, smem, sms, blocks);
    if (rc) return rc;
    void* args[] = {&P};
    cudaError_t e;
    if (gauss) {
        e = ensure_smem_attr((const void*)tl::k_pcg<true>, smem);
        if (e != cudaSuccess) return fail(TL_E_CUDA, cudaGetErrorString(e));
        e = cudaLaunchCooperativeKernel((void*)tl::k_pcg<true>, blocks, tl::kTPB, args, smem, st);
    } else {
        e = cudaLaunchCooperativeKernel((void*)tl::k_pcg<false>, blocks, tl::kTPB, args, smem, st);
    }
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("k_pcg launch: ") + cudaGetErrorString(e));
    if (launches) ++*launches;
    return TL_OK;
}

// ---- streaming PCG in four launches (tl_stream.cuh) ----------------------------------
// Default for grids that do not fit on chip; TLGPU_SPLIT=0 restores the single cooperative
// k_pcg.  TLGPU_SMINB picks the CG loop kernel's CTAs per SM and unroll: 2, 3, 4 (one
// node per trip) or 22, 32 (two); default 32 (40 registers, 1536 threads per SM, measured
// best on the cfg3 / cfg4 grids: profiles/README.md).
static int split_minb() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TLGPU_SPLIT");
        const char* m = getenv("TLGPU_SMINB");
        v = (e && e[0] == '0') ? 0 : (m ? atoi(m) : 32);
        if (v != 0 && v != 2 && v != 3 && v != 4 && v != 22 && v != 32) v = 32;
    }
    return v;
}

template <int MINB, int UNR = 1>
static cudaError_t launch_s_cg(tl::PcgParams& P, int Gr, int sms, cudaStream_t st) {
    static thread_local int per_sm = 0;
    if (per_sm == 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tl::k_s_cg<MINB, UNR>, tl::kSTPB, 0);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
    }
    const int G = per_sm * sms;
    void* args[] = {&P, &Gr};
    return cudaLaunchCooperativeKernel((void*)tl::k_s_cg<MINB, UNR>, G, tl::kSTPB, args, 0, st);
}

// ---- z-marching CG loop on bulk copies (tl_tiled.cuh) --------------------------------
// Default CG loop of the streaming solve; TLGPU_TILED=0 falls back to k_s_cg, and grids
// below TLGPU_TILED_MIN nodes (default 1M) use k_s_cg too.  Item plan: tiled_plan_range.
// consumer warps of k_t_cg: 16 (+ producer = 17 warps) or 19 (20 warps), both at 96 registers;
// the item planner picks per grid (more warps hide more latency, fewer leave less of a
// half-empty second consumer slot on narrow planes)
constexpr int kTNCWs[2] = {16, 19};
static bool tiled_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TLGPU_TILED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static bool tiled_plan_range(const tl::Grid& g, int sms, int zlo, int zhi, tl::TPlan& tp, size_t& smem, int nsys = 1);

// TLGPU_SNAKE=0: both sweeps of the streaming CG loops walk the grid bottom-up (default 1:
// sweep B top-down, L2 reuse across the sweeps; tl_tiled.cuh)
static int snake_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TLGPU_SNAKE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

static bool tiled_plan(const tl::Grid& g, int sms, tl::TPlan& tp, size_t& smem) {
    static long long nmin = -1;
    if (nmin < 0) {
        const char* e = getenv("TLGPU_TILED_MIN");
        nmin = e ? atoll(e) : 1000000LL;
    }
    if ((long long)g.n < nmin) return false;
    return tiled_plan_range(g, sms, 0, g.NZ, tp, smem);
}

// Item plan of the bulk-copy z-march over node planes [zlo, zhi) (the whole grid, or one
// rank's own planes of a z-slab decomposition).
//
// An item is H full x-rows by one z chunk.  The plan minimises a cost model fitted to
// sweeps of the BASELINE grids (tools/tune_snake.sh, tools/sweep_profile.py):
//   cost(H, C) = waves * (Z + o) * plane,   waves = ceil(NB * C / CTAs),  Z = planes / C,  o = 2 or 0.5
//   plane      = max(512 * ceil(H NX / 512), H NX (1 + 0.6 / H))
// - items are taken dynamically but are all about the same size, so a sweep lasts `waves`
//   items per CTA: balance (items a multiple of the CTA count) dominates;
// - an item costs o planes beyond its own (halo plane, pipeline fill, reduction, tail: see below);
// - a plane costs its consumer slots (512 threads take one node each per slot) or its ring
//   traffic including the halo rows, whichever is larger.
// A batched solve (k_tb_cg) sweeps nsys systems of this shape together: its item count is
// nsys times the plan's, so it takes fewer, larger items per system.
// Constraints: H NX <= 2 x 512 nodes per plane where possible (the lean plane loops keep two
// nodes' coefficients per thread in registers; up to 4 x 512 otherwise), at least 4 ring
// stages in 220 KB.  TLGPU_TH / TLGPU_TC / TLGPU_TZ override H, the chunk count and the
// smallest chunk.
static bool tiled_plan_range(const tl::Grid& g, int sms, int zlo, int zhi, tl::TPlan& tp, size_t& smem, int nsys) {
    const int NX = g.NX;
    const int nzr = zhi - zlo;
    if (nzr < 1) return false;
    auto even = [](int v) { return (v + 1) & ~1; };
    const size_t cap = 220 * 1024;
    auto stage_of = [&](int H) {
        const int RA = even((H + 1) * NX + 2), RB = even((H + 2) * NX + 2), RX = even(H * NX + 2);
        return (std::max(2 * RA, RB + 2 * RX) + 15) & ~15;
    };
    auto stages_of = [&](int H) { return (int)std::min<size_t>(tl::kTMaxStages, cap / ((size_t)stage_of(H) * 8)); };
    int zmin = 2;
    if (const char* e = getenv("TLGPU_TZ")) zmin = std::max(1, atoi(e));
    // what an item costs beyond its own planes, in planes: ~2 on grids of a few L2 sizes
    // (halo planes, pipeline fill and drain show with 1-4 items per CTA), ~0.5 on sweeps
    // far larger than L2 (tens of items per CTA: the producer streams the next item while
    // the current one computes; cfg4 global: C = 5 chunks 39.1 ms, C = 1 40.0 ms, C = 13 40.0 ms)
    const double sweep_bytes = 40.0 * (double)NX * g.NY * nzr * nsys;
    const double item_planes = sweep_bytes > 1e9 ? 0.5 : 2.0;
    int want_ncw = 0;
    if (const char* e = getenv("TLGPU_NCW")) want_ncw = atoi(e);
    int H = 0, nch = 0, ncw = 0, Hmax = 0;
    double best = 1e300;
    for (int w = 0; w < 2; ++w) {
        const int nw = kTNCWs[w];
        if (want_ncw && want_ncw != nw) continue;
        const int npt_max = NX <= 2 * nw * 32 ? 2 : 4;
        int hmax = std::min(g.NY, npt_max * nw * 32 / NX);
        while (hmax >= 1 && stages_of(hmax) < 4) --hmax;
        for (int h = 1; h <= hmax; ++h) {
            const int NB = (g.NY + h - 1) / h;
            const int slots = (h * NX + nw * 32 - 1) / (nw * 32);
            const double plane = std::max((double)slots * nw * 32, (double)h * NX * (1.0 + 0.6 / h));
            for (int c = 1; c <= std::min(nzr, tl::kTMaxChunks); ++c) {
                const int Z = (nzr + c - 1) / c;
                if (Z < zmin && c > 1) break;
                const long long I = (long long)NB * c;
                if (I > tl::kTMaxItems) break;
                const long long waves = (I * nsys + sms - 1) / sms;     // nsys: systems of a batched solve
                const double cost = (double)waves * ((double)nzr / c + item_planes) * plane;
                if (cost < best * (1.0 - 1e-9)) { best = cost; H = h; nch = c; ncw = nw; Hmax = hmax; }
            }
        }
    }
    if (H == 0) return false;
    tp.ncw = ncw;
    if (const char* e = getenv("TLGPU_TH")) H = std::max(1, std::min(atoi(e), Hmax));
    if (const char* e = getenv("TLGPU_TC")) nch = std::max(1, std::min(atoi(e), std::min(nzr, tl::kTMaxChunks)));
    tp.H = H;
    tp.NB = (g.NY + H - 1) / H;
    tp.RA = even((H + 1) * NX + 2);
    tp.RB = even((H + 2) * NX + 2);
    tp.RX = even(H * NX + 2);
    tp.stage = stage_of(H);
    tp.NS = stages_of(H);
    if (tp.NS < 4) return false;
    tp.C = nch;
    tp.I = tp.NB * tp.C;
    if (tp.I > tl::kTMaxItems) return false;
    tp.kb[0] = (short)zlo;
    for (int c = 0; c < tp.C; ++c) tp.kb[c + 1] = (short)(zlo + (long long)nzr * (c + 1) / nch);
    tp.nsd.init(tp.NS);
    tp.nbd.init(tp.NB);
    tp.snake = snake_enabled();
    smem = (size_t)tp.NS * tp.stage * 8;
    if (getenv("TLGPU_VERBOSE"))
        fprintf(stderr, "[tlgpu] item plan %dx%dx[%d,%d): H=%d NB=%d C=%d I=%d (%.2f per CTA) NS=%d stage=%d B snake=%d "
                "consumer warps=%d\n",
                g.NX, g.NY, zlo, zhi, tp.H, tp.NB, tp.C, tp.I, (double)tp.I / sms, tp.NS, tp.stage * 8, tp.snake, tp.ncw);
    return true;
}

static unsigned long long* prof_buffer();

static cudaError_t launch_t_cg(tl::PcgParams& P, int Gr, int sms, cudaStream_t st, bool& launched,
                               const tl::TPlan& tp, size_t smem) {
    launched = false;
    const int ncw = tp.ncw;
    // nodes per consumer thread per plane: 1, 2 (lean plane loops) or 4
    const int nodes = tp.H * P.g.NX;
    const int npt = nodes <= ncw * 32 ? 1 : (nodes <= 2 * ncw * 32 ? 2 : 4);
    auto kern = ncw == 16 ? (npt == 1 ? tl::k_t_cg<16, 1> : npt == 2 ? tl::k_t_cg<16, 2> : tl::k_t_cg<16, 4>)
                          : (npt == 1 ? tl::k_t_cg<19, 1> : npt == 2 ? tl::k_t_cg<19, 2> : tl::k_t_cg<19, 4>);
    cudaError_t e = ensure_smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (ncw + 1) * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaSuccess;
    e = cudaMemsetAsync(P.part + tl::kTCounter, 0, 4 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    tl::TPlan tpl = tp;
    tpl.prof = prof_buffer();
    void* args[] = {&P, &Gr, (void*)&tpl};
    e = cudaLaunchCooperativeKernel((void*)kern, sms, (ncw + 1) * 32, args, smem, st);
    launched = e == cudaSuccess;
    return e;
}

static int launch_stream(tl::PcgParams& P, int sms, cudaStream_t st, int64_t* launches) {
    const int minb = split_minb();
    if (minb == 0) return launch_pcg(P, false, sms, st, launches);
    // one resident wave of each pass (a grid larger than what fits leaves a thin second wave)
    static thread_local int occ_rhs = 0, occ_res = 0;
    if (occ_rhs == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_rhs, tl::k_s_rhs, tl::kSTPB, 0) != cudaSuccess || occ_rhs < 1)
            occ_rhs = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_res, tl::k_s_resid, tl::kSTPB, 0) != cudaSuccess || occ_res < 1)
            occ_res = 1;
    }
    const int Gr = std::min(4, occ_rhs) * sms, Gq = std::min(4, occ_res) * sms;
    tl::TPlan tp{};
    size_t smem = 0;
    const bool use_tiled = tiled_enabled() && tiled_plan(P.g, sms, tp, smem);
    // k_t_cg takes r0 = b and x0 = 0 as implied: the RHS writes b only
    P.light_rhs = use_tiled ? 1 : 0;
    P.snake = snake_enabled();
    P.prof = prof_buffer();
    tl::k_s_rhs<<<Gr, tl::kSTPB, 0, st>>>(P);
    cudaError_t e = cudaGetLastError();
    bool tiled = false;
    if (e == cudaSuccess && use_tiled) e = launch_t_cg(P, Gr, sms, st, tiled, tp, smem);
    if (e == cudaSuccess && use_tiled && !tiled) {
        // no k_t_cg after all (occupancy): rebuild the RHS with r0 and x0 written
        P.light_rhs = 0;
        tl::k_s_rhs<<<Gr, tl::kSTPB, 0, st>>>(P);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && !tiled)
        e = minb == 2 ? launch_s_cg<2>(P, Gr, sms, st)
          : minb == 4 ? launch_s_cg<4>(P, Gr, sms, st)
          : minb == 22 ? launch_s_cg<2, 2>(P, Gr, sms, st)
          : minb == 32 ? launch_s_cg<3, 2>(P, Gr, sms, st)
                       : launch_s_cg<3>(P, Gr, sms, st);
    if (e == cudaSuccess) {
        tl::k_s_resid<<<Gq, tl::kSTPB, 0, st>>>(P);
        tl::k_s_final<<<1, tl::kSTPB, 0, st>>>(P, Gq);
        e = cudaGetLastError();
    }
    P.light_rhs = 0;
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("streaming solve launch: ") + cudaGetErrorString(e));
    if (launches) *launches += 4;
    return TL_OK;
}

// ---- SMEM-resident brick PCG: decomposition + launch ------------------------------
// 227 KB of shared memory per CTA on sm_100, minus the kernels' static ClassTable and
// reduction scratch (3.6 KB) and some slack.
static constexpr int kResSmemCap = 232448 - 4096;
struct BrickPlan {
    bool ok = false;
    int ng[3] = {1, 1, 1};
    int maxnodes = 0;
    size_t smem = 0;
    int npt = 0;
    bool xglob = false;          // CG-CG with x in global memory (see rescg_smem_bytes)
};

static void split_axis(int N, int parts, int* off) {
    for (int e = 0; e <= parts; ++e) off[e] = (int)((long long)N * e / parts);
}

static BrickPlan plan_bricks_uncached(const tl::Grid& g, bool gauss, int sms, size_t smem_cap, bool cgv) {
    BrickPlan best;
    const int N[3] = {g.NX, g.NY, g.NZ};
    const long long n = (long long)g.n;
    // small grids: fewer, larger bricks (cheaper barriers); large: one brick per SM
    int target = (int)std::min<long long>(sms, std::max<long long>(1, (n + 2047) / 2048));
    const int gtab = gauss ? tl::gauss_smem_len(g) : 0;
    double best_cost = 1e300;
    // CG-CG: x in SMEM if any decomposition fits, else x in global memory
    for (int xg = 0; xg < ((cgv && gtab == 0) ? 2 : 1) && !best.ok; ++xg)
    for (int gx = 1; gx <= std::min(N[0], tl::kResMaxSplit); ++gx)
        for (int gy = 1; gy <= std::min(N[1], tl::kResMaxSplit) && gx * gy <= target; ++gy)
            for (int gz = 1; gz <= std::min(N[2], tl::kResMaxSplit) && gx * gy * gz <= target; ++gz) {
                const int G = gx * gy * gz;
                if (G > tl::kResMaxBlocks) continue;
                const int lx = (N[0] + gx - 1) / gx, ly = (N[1] + gy - 1) / gy, lz = (N[2] + gz - 1) / gz;
                const int own = lx * ly * lz;
                const int H = (lx + 2) * (ly + 2) * (lz + 2);
                const int nface = 2 * (ly * lz + lx * lz + lx * ly);
                const size_t smem = cgv ? tl::rescg_smem_bytes(lx, ly, lz, gtab, xg == 1)
                                        : tl::res_smem_bytes(lx, ly, lz, gtab);
                if (own > 12 * tl::kResTPB || smem > smem_cap || H >= 16384 ||
                    nface > tl::kResKF * tl::kResTPB)
                    continue;
                // cost: max work per CTA, then halo, then fewer CTAs
                const double cost = (double)own * 1.0 + 0.25 * (double)(H - own) + 0.01 * G;
                if (cost < best_cost) {
                    best_cost = cost;
                    best.ok = true;
                    best.ng[0] = gx; best.ng[1] = gy; best.ng[2] = gz;
                    best.maxnodes = own;
                    best.smem = smem;
                    best.xglob = xg == 1;
                }
            }
    if (best.ok) {
        int npt = (best.maxnodes + tl::kResTPB - 1) / tl::kResTPB;
        best.npt = npt <= 4 ? 4 : npt <= 8 ? 8 : 12;
    }
    return best;
}

// decomposition cache keyed by grid shape (the search is a few hundred microseconds)
static BrickPlan plan_bricks(const tl::Grid& g, bool gauss, int sms, size_t smem_cap, bool cgv) {
    struct Entry { int nc[3]; bool gauss; int sms; bool cgv; BrickPlan plan; };
    static thread_local std::vector<Entry> cache;
    for (const Entry& e : cache)
        if (e.nc[0] == g.nc[0] && e.nc[1] == g.nc[1] && e.nc[2] == g.nc[2] && e.gauss == gauss &&
            e.sms == sms && e.cgv == cgv)
            return e.plan;
    BrickPlan bp = plan_bricks_uncached(g, gauss, sms, smem_cap, cgv);
    cache.push_back({{g.nc[0], g.nc[1], g.nc[2]}, gauss, sms, cgv, bp});
    return bp;
}

// Default: the one-barrier Chronopoulos-Gear kernel wherever its larger SMEM footprint
// fits (the cfg2 local grid: 8.7 us vs 9.5 us per iteration), else the two-barrier kernel
// that mirrors scipy's cg operation for operation.  TLGPU_EXACT_CG=1 forces the latter.
static bool exact_cg() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TLGPU_EXACT_CG");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

template <bool GAUSS, int NPT, bool MULTI, bool XG = false>
static cudaError_t launch_rescg_t(tl::ResCGParams& RP, int G, size_t smem, cudaStream_t st) {
    auto fn = tl::k_pcg_resident_cg<GAUSS, NPT, MULTI, XG>;
    cudaError_t e = ensure_smem_attr((const void*)fn, kResSmemCap);
    if (e != cudaSuccess) return e;
    void* args[] = {&RP};
    return cudaLaunchCooperativeKernel((void*)fn, G, tl::kResTPB, args, smem, st);
}

template <bool GAUSS, bool MULTI = false>
static cudaError_t launch_rescg_g(tl::ResCGParams& RP, int npt, int G, size_t smem, cudaStream_t st) {
    if (RP.xglob) {                  // x in global memory: large bricks, no Gaussian tables
        if (GAUSS || npt < 8) return cudaErrorInvalidConfiguration;
        return npt == 8 ? launch_rescg_t<false, 8, MULTI, true>(RP, G, smem, st)
                        : launch_rescg_t<false, 12, MULTI, true>(RP, G, smem, st);
    }
    switch (npt) {
        case 4: return launch_rescg_t<GAUSS, 4, MULTI>(RP, G, smem, st);
        case 8: return launch_rescg_t<GAUSS, 8, MULTI>(RP, G, smem, st);
        default: return launch_rescg_t<GAUSS, 12, MULTI>(RP, G, smem, st);
    }
}

static unsigned long long* g_prof = nullptr;     // TLGPU_PROF=1: phase timestamps of block 0
constexpr int kProfLen = 8192;                   // [0, 1024) resident kernels; 1024 + 16 b + slot: k_t_cg CTA b

static unsigned long long* prof_buffer() {
    static int want = -1;
    if (want < 0) {
        const char* e = getenv("TLGPU_PROF");
        want = (e && e[0] == '1') ? 1 : 0;
        if (want && cudaMalloc((void**)&g_prof, kProfLen * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(g_prof, 0, kProfLen * sizeof(unsigned long long));
    }
    return g_prof;
}

template <bool GAUSS, int NPT>
static cudaError_t launch_res_t(tl::ResParams& RP, int G, size_t smem, cudaStream_t st) {
    auto fn = tl::k_pcg_resident<GAUSS, NPT>;
    cudaError_t e = ensure_smem_attr((const void*)fn, kResSmemCap);
    if (e != cudaSuccess) return e;
    void* args[] = {&RP};
    return cudaLaunchCooperativeKernel((void*)fn, G, tl::kResTPB, args, smem, st);
}

template <bool GAUSS>
static cudaError_t launch_res_g(tl::ResParams& RP, int npt, int G, size_t smem, cudaStream_t st) {
    switch (npt) {
        case 4: return launch_res_t<GAUSS, 4>(RP, G, smem, st);
        case 8: return launch_res_t<GAUSS, 8>(RP, G, smem, st);
        default: return launch_res_t<GAUSS, 12>(RP, G, smem, st);
    }
}

static int g_force_streaming = -1;

static bool force_streaming() {
    if (g_force_streaming < 0) {
        const char* e = getenv("TLGPU_STREAMING");
        g_force_streaming = (e && e[0] == '1') ? 1 : 0;
    }
    return g_force_streaming == 1;
}

// Resident kernel when the grid fits on-chip, streaming k_pcg otherwise.
// Exchange buffer layout (4 n doubles): [r0 / final x][w ping-pong: 2 n][saved T_old: n].
static void fill_rescg(tl::ResCGParams& RP, const tl::PcgParams& P, double* xg, const BrickPlan& bp) {
    RP.P = P;
    RP.xr = xg;
    RP.xw = xg + P.g.n;
    RP.saved = xg + 3 * (size_t)P.g.n;
    RP.prof = prof_buffer();
    const int N[3] = {P.g.NX, P.g.NY, P.g.NZ};
    for (int a = 0; a < 3; ++a) {
        RP.ng[a] = bp.ng[a];
        split_axis(N[a], bp.ng[a], RP.off[a]);
    }
}

static bool cg_fits(const tl::Grid& g, bool gauss, int sms, BrickPlan& bp) {
    if (force_streaming() || exact_cg()) return false;
    bp = plan_bricks(g, gauss, sms, kResSmemCap, true);
    return bp.ok;
}

// Per-grid cache of the resident CG-CG kernel's static setup (tl_resident_cg.cuh) and its
// tail counter; owned by a tl_run (one per level).
struct ResCache {
    int* buf = nullptr;
    size_t cap = 0;              // ints
    double* xbuf = nullptr;      // own-node x of an xglob plan
    size_t xcap = 0;
    unsigned* counter = nullptr;
    int key[7] = {0, 0, 0, 0, 0, 0, 0};   // grid cells + brick split + npt of the stored setup
    bool ready = false;
    void release() {
        if (buf) cudaFree(buf);
        if (counter) cudaFree(counter);
        if (xbuf) cudaFree(xbuf);
        xbuf = nullptr;
        xcap = 0;
        buf = nullptr;
        counter = nullptr;
        cap = 0;
        ready = false;
    }
};

// Sets RP.scache / sc_mode / tail_count from the cache (allocating it on first use).
static int attach_cache(ResCache* rc, tl::ResCGParams& RP, const tl::Grid& g, const BrickPlan& bp) {
    if (!rc) return TL_OK;
    if (!rc->counter) {
        TL_CUDA(cudaMalloc((void**)&rc->counter, 2 * sizeof(unsigned)));   // tail, barrier
        TL_CUDA(cudaMemset(rc->counter, 0, 2 * sizeof(unsigned)));
    }
    RP.tail_count = rc->counter;
    const char* cb = getenv("TLGPU_CGSYNC");          // 1: cg grid.sync in the CG loop
    const int Gb = bp.ng[0] * bp.ng[1] * bp.ng[2];
    RP.bar_count = ((cb && cb[0] == '1') || Gb > 160) ? nullptr : rc->counter + 1;   // grid_allreduce: G <= 160
    long long stride = 0;
    for (int bz = 0; bz < bp.ng[2]; ++bz)
        for (int by = 0; by < bp.ng[1]; ++by)
            for (int bx = 0; bx < bp.ng[0]; ++bx) {
                const int lx = RP.off[0][bx + 1] - RP.off[0][bx], ly = RP.off[1][by + 1] - RP.off[1][by];
                const int lz = RP.off[2][bz + 1] - RP.off[2][bz];
                const long long H = (long long)(lx + 2) * (ly + 2) * (lz + 2);
                const long long nf = 2LL * (ly * lz + lx * lz + lx * ly);
                const long long need = (H + 3) / 4 + 2 * nf + (long long)lx * ly * lz + (long long)bp.npt * tl::kResTPB;
                stride = std::max(stride, need);
            }
    const int G = bp.ng[0] * bp.ng[1] * bp.ng[2];
    const int key[7] = {g.nc[0], g.nc[1], g.nc[2], bp.ng[0], bp.ng[1], bp.ng[2], bp.npt};
    const size_t want = (size_t)stride * G;
    if (want > rc->cap) {
        if (rc->buf) cudaFree(rc->buf);
        rc->buf = nullptr;
        TL_CUDA(cudaMalloc((void**)&rc->buf, want * sizeof(int)));
        rc->cap = want;
        rc->ready = false;
    }
    if (!std::equal(key, key + 7, rc->key)) {
        std::copy(key, key + 7, rc->key);
        rc->ready = false;
    }
    RP.scache = rc->buf;
    RP.sc_stride = stride;
    RP.sc_mode = rc->ready ? 2 : 1;
    if (bp.xglob) {
        const size_t xn = (size_t)bp.maxnodes * G;
        if (xn > rc->xcap) {
            if (rc->xbuf) cudaFree(rc->xbuf);
            rc->xbuf = nullptr;
            TL_CUDA(cudaMalloc((void**)&rc->xbuf, xn * sizeof(double)));
            rc->xcap = xn;
        }
        RP.xglob = rc->xbuf;
        RP.xg_stride = bp.maxnodes;
    }
    return TL_OK;
}

static int launch_solve(tl::PcgParams& P, bool gauss, int sms, double* xg, cudaStream_t st,
                        int64_t* launches, tl::SolveSpec* dspec = nullptr, int* kind_out = nullptr,
                        ResCache* cache = nullptr) {
    BrickPlan bp;
    if (xg && dspec && cg_fits(P.g, gauss, sms, bp) && (!bp.xglob || (cache && !getenv("TLGPU_NOCACHE")))) {
        {
            tl::SolveSpec hs{};
            hs.mbase = P.mbase;
            hs.w = P.w;
            hs.src = P.src;
            hs.src.on = gauss ? 1 : 0;
            hs.tin = 0;
            hs.save_before = 0;
            hs.tout = 1;
            hs.info = P.info;
            hs.snap = nullptr;
            tl::ResCGParams RP{};
            fill_rescg(RP, P, xg, bp);
            RP.specs = nullptr;          // the spec travels in the kernel parameters
            RP.spec0 = hs;
            RP.nspec = 1;
            if (getenv("TLGPU_NOCACHE") == nullptr)
                if (int rc = attach_cache(cache, RP, P.g, bp)) return rc;
            const int G = bp.ng[0] * bp.ng[1] * bp.ng[2];
            cudaError_t e = gauss ? launch_rescg_g<true>(RP, bp.npt, G, bp.smem, st)
                                  : launch_rescg_g<false>(RP, bp.npt, G, bp.smem, st);
            if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("k_pcg_resident_cg launch: ") + cudaGetErrorString(e));
            if (launches) ++*launches;
            if (kind_out) *kind_out = 2;
            if (RP.scache) cache->ready = true;
            return TL_OK;
        }
    }
    if (xg && !force_streaming()) {
        BrickPlan bp = plan_bricks(P.g, gauss, sms, 200 * 1024, false);
        if (bp.ok) {
            tl::ResParams RP{};
            RP.P = P;
            RP.xg = xg;              // exchange buffer holds 4 n doubles: r, x, q (x2)
            RP.xx = xg + P.g.n;
            RP.prof = prof_buffer();
            const int N[3] = {P.g.NX, P.g.NY, P.g.NZ};
            for (int a = 0; a < 3; ++a) {
                RP.ng[a] = bp.ng[a];
                split_axis(N[a], bp.ng[a], RP.off[a]);
            }
            const int G = bp.ng[0] * bp.ng[1] * bp.ng[2];
            cudaError_t e = gauss ? launch_res_g<true>(RP, bp.npt, G, bp.smem, st)
                                  : launch_res_g<false>(RP, bp.npt, G, bp.smem, st);
            if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("k_pcg_resident launch: ") + cudaGetErrorString(e));
            if (launches) ++*launches;
            if (kind_out) *kind_out = 1;
            return TL_OK;
        }
    }
    if (kind_out) *kind_out = 0;
    if (gauss && xg && P.load == nullptr) {
        // streaming path: Gaussian load into the second half of the exchange buffer by a
        // plain kernel, then the lean (non-Gaussian) cooperative solve adds it
        double* gl = xg + P.g.n;
        const size_t smem = gauss_smem(P.g);
        TL_CUDA(ensure_smem_attr((const void*)tl::k_gauss_load, smem));
        tl::k_gauss_load<<<2 * sms, 256, smem, st>>>(P.g, P.src, P.mbase, P.T, gl);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("k_gauss_load: ") + cudaGetErrorString(e));
        if (launches) ++*launches;
        P.load = gl;
        return launch_stream(P, sms, st, launches);
    }
    if (!gauss) return launch_stream(P, sms, st, launches);
    return launch_pcg(P, gauss, sms, st, launches);
}

void set_coeffs(tl::PcgParams& P, double kappa, double rho_c, double dt) {
    const double V = P.g.h[0] * P.g.h[1] * P.g.h[2];
    for (int a = 0; a < 3; ++a) P.cbase[a] = kappa * V / (P.g.h[a] * P.g.h[a]) / 6.0;
    P.mbase = (rho_c / dt) * V / 24.0;
}

int device_sms(int dev, int& sms) {
    TL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return TL_OK;
}

template <class T>
int dalloc(T** p, size_t n) {
    // +2 elements: the bulk copies of k_t_cg round node ranges out to 16-byte boundaries
    cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (n + 2));
    if (e != cudaSuccess) return fail(TL_E_ALLOC, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return TL_OK;
}

}  // namespace

struct tl_run {
    int device = 0, sms = 0;
    cudaStream_t stream = nullptr;
    tl_run_desc desc{};
    tl::Grid G{}, L{};
    double* Tg = nullptr; double* bg = nullptr; double* rg = nullptr; double* pg0 = nullptr; double* pg1 = nullptr; double* qg = nullptr;
    double* loadg = nullptr;
    double* Tl = nullptr; double* bl = nullptr; double* rl = nullptr; double* pl0 = nullptr; double* pl1 = nullptr; double* ql = nullptr;
    double* tr_old = nullptr; double* tr_pred = nullptr; double* Tl_before = nullptr;
    double* part = nullptr;
    int* dep_prev = nullptr; int* dep_prev_n = nullptr;
    double* dep_pts = nullptr; double* dep_pow = nullptr; int dep_cap = 0;
    tl::SolveInfoDev* info = nullptr; int info_cap = 0; int info_n = 0;
    double* melt = nullptr; double* melt_part = nullptr; double* melt_host = nullptr;
    double* snap_g = nullptr; std::vector<double*> snap_l; int snap_n = 0;
    double* xg = nullptr;            // exchange array of the resident kernels (4 n)
    void* gather_buf = nullptr; size_t gather_cap = 0;     // tl_run_get_field_at scratch
    void* batch_dev = nullptr;       // batched solves led by this run: parameter buffer, sweep counters
    unsigned* batch_ctr = nullptr;
    tl::SolveSpec* d_specs = nullptr; int specs_cap = 0;
    ResCache cache_g, cache_l;       // resident-kernel setup caches (global / local grid)
    // asynchronous field read-back (tl_run_field_async): staging copies + copy stream
    cudaStream_t copy_stream = nullptr;
    double* stage[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t stage_n[4] = {0, 0, 0, 0};
    cudaEvent_t stage_ready[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t stage_done[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<tl::SolveSpec> h_specs;
    std::vector<int> ev_nsolve;
    double* flush = nullptr; size_t flush_n = 0;
    double* gload = nullptr; tl::Gauss* d_srcs = nullptr; int gload_cap = 0;   // multi-solve Gaussian loads
    std::vector<tl::Gauss> h_srcs;
    int64_t launches = 0;
    bool external_global = false;   // global field supplied by the slab solve (multi-GPU)
    int ext_k0 = 0;                 // external mode: first stored global plane
    double* Tg_store = nullptr;     // external mode: planes [ext_k0, NZ); Tg = Tg_store - ext_k0 nxy
    bool timing = false;
    std::vector<cudaEvent_t> ev;     // pairs
    std::vector<int> ev_level;
    int ev_n = 0;                    // pairs in use
};

static int timed_begin(tl_run* R, int level, int nsolve = 1) {
    if (!R->timing) return TL_OK;
    while ((int)R->ev.size() < 2 * (R->ev_n + 1)) {
        cudaEvent_t e;
        TL_CUDA(cudaEventCreate(&e));
        R->ev.push_back(e);
    }
    if ((int)R->ev_level.size() < R->ev_n + 1) R->ev_level.resize(R->ev_n + 1);
    R->ev_level[R->ev_n] = level;
    if ((int)R->ev_nsolve.size() < R->ev_n + 1) R->ev_nsolve.resize(R->ev_n + 1);
    R->ev_nsolve[R->ev_n] = nsolve;
    TL_CUDA(cudaEventRecord(R->ev[2 * R->ev_n], R->stream));
    return TL_OK;
}

static int timed_end(tl_run* R) {
    if (!R->timing) return TL_OK;
    TL_CUDA(cudaEventRecord(R->ev[2 * R->ev_n + 1], R->stream));
    ++R->ev_n;
    return TL_OK;
}

extern "C" {

int32_t tl_abi_version(void) { return TLGPU_ABI_VERSION; }

const char* tl_last_error(void) { return g_err.c_str(); }

int32_t tl_device_query(int32_t device, int32_t* sm_count, int64_t* l2_bytes, int32_t* coop) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) return fail(TL_E_NODEVICE, "no CUDA device");
    int v = 0;
    TL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    if (sm_count) *sm_count = v;
    TL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device));
    if (l2_bytes) *l2_bytes = v;
    TL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, device));
    if (coop) *coop = v;
    return TL_OK;
}

// ------------------------------------------------------------------------------------
// Single step on host buffers (seam 3: fem.step_backward_euler for a linear problem).
// ------------------------------------------------------------------------------------
static float g_step_last_ms = 0.0f;

int32_t tl_step_last_ms(float* ms) {
    if (!ms) return fail(TL_E_INVALID, "null argument");
    *ms = g_step_last_ms;
    return TL_OK;
}

static int step_impl(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                     int32_t dirichlet_kind, const double* gA, const double* gB, double w,
                     double g_const, const double* T_old, const double* load,
                     const tl_gaussian* src, double rtol, int32_t maxiter, double* x_out,
                     tl_solve_info* info, const int32_t* dnodes, int64_t nd, const double* dvalues);

int32_t tl_step_host(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                     int32_t dirichlet_kind, const double* gA, const double* gB, double w,
                     double g_const, const double* T_old, const double* load,
                     const tl_gaussian* src, double rtol, int32_t maxiter, double* x_out,
                     tl_solve_info* info) {
    return step_impl(grid, kappa, rho_c, dt, dirichlet_kind, gA, gB, w, g_const, T_old, load, src, rtol, maxiter,
                     x_out, info, nullptr, 0, nullptr);
}

int32_t tl_step_nodes_host(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                           int32_t dirichlet_kind, const int32_t* dirichlet_nodes, int64_t n_dirichlet,
                           const double* dirichlet_values, const double* T_old, const double* load,
                           const tl_gaussian* src, double rtol, int32_t maxiter, double* x_out,
                           tl_solve_info* info) {
    if (n_dirichlet < 0 || (n_dirichlet > 0 && (!dirichlet_nodes || !dirichlet_values)))
        return fail(TL_E_INVALID, "Dirichlet node list");
    return step_impl(grid, kappa, rho_c, dt, dirichlet_kind, nullptr, nullptr, 0.0, 0.0, T_old, load, src, rtol,
                     maxiter, x_out, info, dirichlet_nodes, n_dirichlet, dirichlet_values);
}

static int step_impl(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                     int32_t dirichlet_kind, const double* gA, const double* gB, double w,
                     double g_const, const double* T_old, const double* load,
                     const tl_gaussian* src, double rtol, int32_t maxiter, double* x_out,
                     tl_solve_info* info, const int32_t* dnodes, int64_t nd, const double* dvalues) {
    if (!grid || !T_old || !x_out) return fail(TL_E_INVALID, "null argument");
    if (dt <= 0) return fail(TL_E_INVALID, "time step must be positive");
    if (dirichlet_kind != tl::kBottom && dirichlet_kind != tl::kGamma)
        return fail(TL_E_INVALID, "unknown Dirichlet kind");
    int dev = 0;
    TL_CUDA(cudaGetDevice(&dev));
    int sms = 0;
    if (int rc = device_sms(dev, sms)) return rc;
    tl::PcgParams P{};
    if (int rc = make_grid(*grid, dirichlet_kind, P.g)) return rc;
    const int n = P.g.n;
    set_coeffs(P, kappa, rho_c, dt);
    const size_t nb = sizeof(double) * n;
    // device workspace kept across calls (the step-level drivers call this once per solve);
    // one per device, grown on demand, calls serialised.  Sub-arrays start on 256-byte
    // boundaries and carry the 2-element tail the bulk-copy CG loop may touch.
    struct StepWs {
        double* ws = nullptr;
        size_t cap = 0;
        cudaStream_t st = nullptr;      // the step's own stream: no device-wide synchronisation
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // solve launch timing (tl_step_last_ms)
    };
    static StepWs wss[64];
    static std::mutex ws_mu;
    std::lock_guard<std::mutex> lock(ws_mu);
    if (dev < 0 || dev >= 64) return fail(TL_E_INVALID, "device ordinal out of range");
    StepWs& W = wss[dev];
    const size_t per = ((size_t)n + 2 + 31) / 32 * 32;
    const size_t npart = tl::kPartLen;
    const size_t nspec = (sizeof(tl::SolveSpec) + sizeof(tl::SolveInfoDev) + 255) / 256 * 32;
    const size_t pnd = dnodes ? ((size_t)nd + 2 + 31) / 32 * 32 : 0;      // node list (ints) + values
    const size_t want = 13 * per + npart + nspec + 2 * pnd;
    if (want > W.cap) {
        if (W.ws) cudaFree(W.ws);
        W.ws = nullptr;
        W.cap = 0;
        TL_CUDA(cudaMalloc((void**)&W.ws, sizeof(double) * want));
        W.cap = want;
    }
    if (!W.st) TL_CUDA(cudaStreamCreateWithFlags(&W.st, cudaStreamNonBlocking));
    cudaStream_t st = W.st;
    double* T = W.ws;
    double* b = W.ws + per;
    double* r = W.ws + 2 * per;
    double* p0 = W.ws + 3 * per;
    double* p1 = W.ws + 4 * per;
    double* q = W.ws + 5 * per;
    double* dA = (gA || dnodes) ? W.ws + 6 * per : nullptr;
    double* dB = gA ? W.ws + 7 * per : dA;
    double* dload = load ? W.ws + 8 * per : nullptr;
    double* xg = W.ws + 9 * per;                       // 4 per
    double* part = W.ws + 13 * per;
    tl::SolveSpec* dspec = reinterpret_cast<tl::SolveSpec*>(W.ws + 13 * per + npart);
    tl::SolveInfoDev* dinfo = reinterpret_cast<tl::SolveInfoDev*>(
        reinterpret_cast<char*>(dspec) + (sizeof(tl::SolveSpec) + 15) / 16 * 16);
    int rc = 0;
    TL_CUDA(copy_in(T, T_old, nb, st, true));
    if (gA) {
        TL_CUDA(copy_in(dA, gA, nb, st, true));
        if (gB && gB != gA) TL_CUDA(copy_in(dB, gB, nb, st, true));
        else dB = dA;
    } else if (dnodes) {
        // Dirichlet data as a node list: the dense array is built on the device
        double* dvl = W.ws + 13 * per + npart + nspec;
        int* dnd = reinterpret_cast<int*>(dvl + pnd);
        TL_CUDA(cudaMemsetAsync(dA, 0, nb, st));
        if (nd > 0) {
            TL_CUDA(copy_in(dnd, dnodes, sizeof(int) * (size_t)nd, st, true));
            TL_CUDA(copy_in(dvl, dvalues, sizeof(double) * (size_t)nd, st, true));
            tl::k_scatter_dirichlet<<<296, 256, 0, st>>>(dnd, dvl, (int)nd, n, nullptr, dA);
            TL_CUDA(cudaGetLastError());
        }
    }
    if (load) TL_CUDA(copy_in(dload, load, nb, st, true));
    P.T = T; P.gA = dA; P.gB = dB; P.w = gA ? w : 0.0; P.g_const = g_const; P.load = dload;
    P.b = b; P.r = r; P.p0 = p0; P.p1 = p1; P.q = q; P.part = part;
    P.rtol = rtol; P.maxiter = maxiter; P.info = dinfo;
    bool gauss = src && src->on;
    if (gauss) {
        P.src.peak = src->peak; P.src.radius = src->radius; P.src.depth = src->depth;
        for (int a = 0; a < 3; ++a) P.src.center[a] = src->center[a];
        P.src.on = 1;
    }
    if (!W.ev0) {
        TL_CUDA(cudaEventCreate(&W.ev0));
        TL_CUDA(cudaEventCreate(&W.ev1));
    }
    TL_CUDA(cudaEventRecord(W.ev0, st));
    rc = launch_solve(P, gauss, sms, xg, st, nullptr, dspec);
    if (rc) return rc;
    TL_CUDA(cudaEventRecord(W.ev1, st));
    tl::SolveInfoDev hi{};
    TL_CUDA(cudaMemcpyAsync(&hi, dinfo, sizeof(hi), cudaMemcpyDeviceToHost, st));
    if (!on_device(x_out)) g_d2h_bytes += (long long)nb;
    TL_CUDA(cudaMemcpyAsync(x_out, T, nb, cudaMemcpyDefault, st));
    TL_CUDA(cudaStreamSynchronize(st));
    TL_CUDA(cudaEventElapsedTime(&g_step_last_ms, W.ev0, W.ev1));
    if (info) {
        info->iterations = hi.iterations; info->status = hi.status; info->bnorm = hi.bnorm;
        info->rnorm = hi.rnorm; info->true_resid = hi.true_resid;
    }
    return TL_OK;
}

static std::mutex g_scratch_mu;
static int scratch(int slot, size_t bytes, void** out);

// Carve `k` device arrays out of scratch slot 3 (256-byte aligned sub-ranges, +2 elements
// each as dalloc gives); the caller holds g_scratch_mu for the whole call.
struct Carve {
    size_t n;
    size_t elem;
    void** out;
};
static int scratch_arrays(std::initializer_list<Carve> arrs) {
    size_t total = 0;
    for (const Carve& c : arrs) total += ((c.n + 2) * c.elem + 255) / 256 * 256;
    void* base = nullptr;
    if (int rc = scratch(3, std::max<size_t>(total, 256), &base)) return rc;
    char* p = static_cast<char*>(base);
    for (const Carve& c : arrs) {
        *c.out = p;
        p += ((c.n + 2) * c.elem + 255) / 256 * 256;
    }
    return TL_OK;
}

int32_t tl_interpolate_host(const tl_grid_desc* global_grid, const double* values,
                            const tl_grid_desc* target, int32_t gamma_only, double* out) {
    if (!global_grid || !values || !target || !out) return fail(TL_E_INVALID, "null argument");
    tl::Grid G{}, L{};
    if (int rc = make_grid(*global_grid, tl::kBottom, G, true)) return rc;
    if (int rc = make_grid(*target, tl::kGamma, L, true)) return rc;
    if (tl::grid_is_2d(G) != tl::grid_is_2d(L)) return fail(TL_E_INVALID, "grids of different dimension");
    double *dv, *dout;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)G.n, 8, (void**)&dv}, {(size_t)L.n, 8, (void**)&dout}})) return rc;
    TL_CUDA(copy_in(dv, values, sizeof(double) * G.n));
    TL_CUDA(copy_in(dout, out, sizeof(double) * L.n));
    if (tl::grid_is_2d(G))
        tl::k_interp2<<<296, 256>>>(G, L, dv, dout, gamma_only ? 1 : 0);
    else
    tl::k_interp<<<592, 256>>>(G, dv, L, gamma_only ? 1 : 0, gamma_only ? nullptr : dout,
                               gamma_only ? dout : nullptr);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(out, dout, sizeof(double) * L.n));
    return TL_OK;
}

static float g_vc_last_ms = 0.0f;

int32_t tl_vc_step_region_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                               const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                               const double* T_lag, const double* extra_load, const tl_gaussian* src,
                               const tl_robin* robin, const uint8_t* dirichlet_mask, const double* g, double rtol,
                               int32_t maxiter, double* x_out, tl_solve_info* info);

int32_t tl_vc_last_cg_ms(float* ms) {
    if (!ms) return fail(TL_E_INVALID, "null argument");
    *ms = g_vc_last_ms;
    return TL_OK;
}

int32_t tl_vc_step_host(const tl_grid_desc* grid, const tl_vc_material* mat, double dt, const double* T_old,
                        const double* T_lag, const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                        const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, double* x_out,
                        tl_solve_info* info) {
    return tl_vc_step_region_host(grid, mat, nullptr, nullptr, 0, dt, T_old, T_lag, extra_load, src, robin,
                                  dirichlet_mask, g, rtol, maxiter, x_out, info);
}

static int vc_impl(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                   const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                   const double* T_lag, const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                   const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, int32_t linear,
                   double picard_tol, int32_t picard_max, double* x_out, int32_t* passes, int32_t* pass_iters,
                   float* pass_ms, double* inc_out, tl_solve_info* info,
                   const int32_t* dnodes = nullptr, int64_t nd = 0, const double* dvalues = nullptr);

int32_t tl_vc_step_region_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                               const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                               const double* T_lag, const double* extra_load, const tl_gaussian* src,
                               const tl_robin* robin, const uint8_t* dirichlet_mask, const double* g, double rtol,
                               int32_t maxiter, double* x_out, tl_solve_info* info) {
    if (!T_lag) return fail(TL_E_INVALID, "null argument");
    int32_t passes = 0, it = 0;
    float ms = 0.0f;
    double inc = 0.0;
    return vc_impl(grid, mat, mat_outside, region, latent_inside_only, dt, T_old, T_lag, extra_load, src, robin,
                   dirichlet_mask, g, rtol, maxiter, 1, 0.0, 1, x_out, &passes, &it, &ms, &inc, info);
}

int32_t tl_vc_picard_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                          const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                          const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                          const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, int32_t linear,
                          double picard_tol, int32_t picard_max, double* x_out, int32_t* passes, int32_t* pass_iters,
                          float* pass_ms, double* inc_out, tl_solve_info* info) {
    if (!passes || !pass_iters || !pass_ms || !inc_out || picard_max < 1) return fail(TL_E_INVALID, "bad argument");
    return vc_impl(grid, mat, mat_outside, region, latent_inside_only, dt, T_old, T_old, extra_load, src, robin,
                   dirichlet_mask, g, rtol, maxiter, linear, picard_tol, picard_max, x_out, passes, pass_iters,
                   pass_ms, inc_out, info);
}

int32_t tl_vc_picard_nodes_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                                const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                                const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                                const int32_t* dirichlet_nodes, int64_t n_dirichlet, const double* dirichlet_values,
                                double rtol, int32_t maxiter, int32_t linear, double picard_tol, int32_t picard_max,
                                double* x_out, int32_t* passes, int32_t* pass_iters, float* pass_ms, double* inc_out,
                                tl_solve_info* info) {
    if (!passes || !pass_iters || !pass_ms || !inc_out || picard_max < 1) return fail(TL_E_INVALID, "bad argument");
    return vc_impl(grid, mat, mat_outside, region, latent_inside_only, dt, T_old, T_old, extra_load, src, robin,
                   nullptr, nullptr, rtol, maxiter, linear, picard_tol, picard_max, x_out, passes, pass_iters,
                   pass_ms, inc_out, info, dirichlet_nodes, n_dirichlet, dirichlet_values);
}

static int vc_impl(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                   const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                   const double* T_lag, const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                   const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, int32_t linear,
                   double picard_tol, int32_t picard_max, double* x_out, int32_t* passes, int32_t* pass_iters,
                   float* pass_ms, double* inc_out, tl_solve_info* info,
                   const int32_t* dnodes, int64_t nd, const double* dvalues) {
    if ((mat_outside || latent_inside_only) && !region) return fail(TL_E_INVALID, "region box required");
    if (mat_outside && (mat_outside->nk < 2 || mat_outside->nc < 2))
        return fail(TL_E_INVALID, "material tables need two rows");
    if (!grid || !mat || !T_old || !T_lag || !x_out || !info) return fail(TL_E_INVALID, "null argument");
    if (dirichlet_mask ? !g : (nd < 0 || (nd > 0 && (!dnodes || !dvalues))))
        return fail(TL_E_INVALID, "Dirichlet data: a mask with values, or a node list with values");
    if (!(dt > 0.0)) return fail(TL_E_INVALID, "time step must be positive");
    if (mat->nk < 2 || mat->nc < 2) return fail(TL_E_INVALID, "material tables need two rows");
    tl::Grid G{};
    if (int rc = make_grid(*grid, tl::kBottom, G, true)) return rc;
    const int n = G.n;
    constexpr int kNB = 296, kT = 256;
    // device workspace kept across calls (a Picard loop calls this once per pass); grown on
    // demand, one per device, calls serialised per process (the workspace is shared)
    struct VcWs {
        double* ws = nullptr;
        size_t cap = 0;
        unsigned char* dm = nullptr;
        size_t dm_cap = 0;              // the mask grows with n, not with `want`
        tl::SolveInfoDev* dinfo = nullptr;
    };
    static VcWs wss[64];
    static std::mutex ws_mu;
    std::lock_guard<std::mutex> lock(ws_mu);
    int cur_dev = 0;
    TL_CUDA(cudaGetDevice(&cur_dev));
    if (cur_dev < 0 || cur_dev >= 64) return fail(TL_E_INVALID, "device ordinal out of range");
    VcWs& W = wss[cur_dev];
    double*& ws = W.ws;
    size_t& ws_cap = W.cap;
    unsigned char*& dm = W.dm;
    tl::SolveInfoDev*& dinfo = W.dinfo;
    double* tabs = nullptr;
    double* cpart = nullptr;
    const size_t per = (size_t)n + 2, nt_i = 2 * (size_t)(mat->nk + mat->nc);
    const size_t nt = nt_i + (mat_outside ? 2 * (size_t)(mat_outside->nk + mat_outside->nc) : 0);
    const bool two_d = tl::grid_is_2d(G);
    const size_t ntet = two_d ? 2 * (size_t)G.nc[0] * G.nc[1] : 6 * (size_t)G.nc[0] * G.nc[1] * G.nc[2];
    const size_t want = 16 * per + nt + 6 * 4096 + 9 * ntet + 2 * ((size_t)nd + 4);
    if (want > ws_cap) {
        if (ws) cudaFree(ws);
        ws = nullptr;
        ws_cap = 0;
        TL_CUDA(cudaMalloc((void**)&ws, sizeof(double) * want));
        ws_cap = want;
    }
    if (per > W.dm_cap) {
        if (dm) cudaFree(dm);
        dm = nullptr;
        W.dm_cap = 0;
        TL_CUDA(cudaMalloc((void**)&dm, per));
        W.dm_cap = per;
    }
    if (!dinfo) TL_CUDA(cudaMalloc((void**)&dinfo, sizeof(tl::SolveInfoDev)));
    double* dTo = ws;
    double* dTl = ws + per;
    double* dex = extra_load ? ws + 2 * per : nullptr;
    double* dg = ws + 3 * per;
    double* diag = ws + 4 * per;
    double* wx = ws + 5 * per;
    double* wy = ws + 6 * per;
    double* wz = ws + 7 * per;
    double* b = ws + 8 * per;
    double* x = ws + 9 * per;
    double* r = ws + 10 * per;
    double* z = ws + 11 * per;
    double* pv = ws + 12 * per;
    double* q = ws + 14 * per;
    tabs = ws + 16 * per;                 // p (ws + 12 per) is a ping-pong pair: 12-13, q at 14
    cpart = tabs + nt;
    double* tk = cpart + 6 * 4096;
    double* tml = tk + ntet;
    double* tsrc = tml + 4 * ntet;
    TL_CUDA(copy_in(dTo, T_old, sizeof(double) * n));
    if (T_lag == T_old) TL_CUDA(cudaMemcpy(dTl, dTo, sizeof(double) * n, cudaMemcpyDeviceToDevice));
    else TL_CUDA(copy_in(dTl, T_lag, sizeof(double) * n));
    if (dex) TL_CUDA(copy_in(dex, extra_load, sizeof(double) * n));
    if (dirichlet_mask) {
        TL_CUDA(copy_in(dg, g, sizeof(double) * n));
        TL_CUDA(copy_in(dm, dirichlet_mask, n));
    } else {
        // sparse Dirichlet data: node list + values, scattered on the device
        int* dnd = reinterpret_cast<int*>(tsrc + 4 * ntet);
        double* dvl = reinterpret_cast<double*>(dnd + ((size_t)nd + 2) / 2 * 2);
        TL_CUDA(cudaMemset(dg, 0, sizeof(double) * n));
        TL_CUDA(cudaMemset(dm, 0, n));
        if (nd > 0) {
            TL_CUDA(copy_in(dnd, dnodes, sizeof(int) * (size_t)nd));
            TL_CUDA(copy_in(dvl, dvalues, sizeof(double) * (size_t)nd));
            tl::k_scatter_dirichlet<<<kNB, kT>>>(dnd, dvl, (int)nd, n, dm, dg);
            TL_CUDA(cudaGetLastError());
        }
    }
    TL_CUDA(cudaMemcpy(tabs, mat->k_T, sizeof(double) * mat->nk, cudaMemcpyHostToDevice));
    TL_CUDA(cudaMemcpy(tabs + mat->nk, mat->k_v, sizeof(double) * mat->nk, cudaMemcpyHostToDevice));
    TL_CUDA(cudaMemcpy(tabs + 2 * mat->nk, mat->c_T, sizeof(double) * mat->nc, cudaMemcpyHostToDevice));
    TL_CUDA(cudaMemcpy(tabs + 2 * mat->nk + mat->nc, mat->c_v, sizeof(double) * mat->nc, cudaMemcpyHostToDevice));
    tl::VcMat M{tabs, tabs + mat->nk, tabs + 2 * mat->nk, tabs + 2 * mat->nk + mat->nc, mat->nk, mat->nc,
                mat->rho, mat->chi, mat->S, mat->T_melt, mat->latent};
    tl::VcMat Mo = M;
    tl::VcRegion RG{};
    if (region) {
        for (int a2 = 0; a2 < 3; ++a2) { RG.lo[a2] = region[a2]; RG.hi[a2] = region[3 + a2]; }
        RG.latent_inside = latent_inside_only ? 1 : 0;
    }
    if (mat_outside) {
        double* t2 = tabs + nt_i;
        const tl_vc_material* m = mat_outside;
        TL_CUDA(cudaMemcpy(t2, m->k_T, sizeof(double) * m->nk, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(t2 + m->nk, m->k_v, sizeof(double) * m->nk, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(t2 + 2 * m->nk, m->c_T, sizeof(double) * m->nc, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(t2 + 2 * m->nk + m->nc, m->c_v, sizeof(double) * m->nc, cudaMemcpyHostToDevice));
        Mo = tl::VcMat{t2, t2 + m->nk, t2 + 2 * m->nk, t2 + 2 * m->nk + m->nc, m->nk, m->nc,
                       m->rho, m->chi, m->S, m->T_melt, m->latent};
        RG.piecewise = 1;
    }
    tl::Gauss S{};
    if (src && src->on) {
        S.peak = src->peak; S.radius = src->radius; S.depth = src->depth;
        for (int a = 0; a < 3; ++a) S.center[a] = src->center[a];
        S.on = 1;
    }
    tl::VcRobin RB{0.0, 0.0, 0.0, 0};
    if (robin && robin->on) RB = tl::VcRobin{robin->h_conv, robin->sigma_eps, robin->T_ambient, 1};
    double inc = INFINITY, prev_inc = INFINITY, theta = 1.0;
    *passes = 0;
    for (int pit = 1; pit <= picard_max; ++pit) {
    if (two_d) {
        tl::k_vc_tris<<<4 * kNB, kT>>>(G, M, Mo, RG, dTo, dTl, dt, S, tk, tml, tsrc);
        tl::k_vc_assemble2<<<kNB, kT>>>(G, tk, tml, tsrc, dTo, dTl, dex, RB, diag, wx, wy, wz, b);
    } else {
    tl::k_vc_tets<<<4 * kNB, kT, sizeof(double) * nt>>>(G, M, Mo, RG, dTo, dTl, dt, S, tk, tml, tsrc);
    tl::k_vc_assemble<<<kNB, kT>>>(G, tk, tml, tsrc, dTo, dTl, dex, RB, diag, wx, wy, wz, b);
    }
    tl::k_vc_constrain_b<<<kNB, kT>>>(G, dm, dg, wx, wy, wz, diag, b);
    tl::k_vc_constrain_w<<<kNB, kT>>>(G, dm, wx, wy, wz);
    TL_CUDA(cudaGetLastError());
    // solve_linear cg branch (fem.py:271-291) with scipy's recurrences: one cooperative launch
    static int per_sm = 0;
    if (per_sm == 0) TL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tl::k_vc_cg, kT, 0));
    int dev = 0, sms = 0;
    TL_CUDA(cudaGetDevice(&dev));
    TL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // blocks per SM of the cooperative PCG: fewer blocks make the two grid barriers and the
    // per-block fixed-order sums of the NB partials cheaper (TLGPU_VC_BPS overrides)
    static int bps = -1;
    if (bps < 0) {
        const char* e = getenv("TLGPU_VC_BPS");
        bps = e ? std::max(1, atoi(e)) : 4;          // measured on 520k nodes: 1: 10.7, 2: 8.3, 4: 7.9, 8: 8.1 ms per step
    }
    const int use_bps = std::min(bps, per_sm);
    const int NBc = std::max(1, std::min(use_bps * sms, (n + kT - 1) / kT));
    if (NBc > 4096) return fail(TL_E_INVALID, "too many CTAs for the reduction workspace");
    tl::VcCg C{diag, wx, wy, wz, b, dm, dg, x, r, z, pv, q, cpart, rtol, maxiter, dinfo};
    void* args[] = {&G, &C};
    cudaEvent_t e0, e1;
    TL_CUDA(cudaEventCreate(&e0));
    TL_CUDA(cudaEventCreate(&e1));
    TL_CUDA(cudaEventRecord(e0, 0));
    TL_CUDA(cudaLaunchCooperativeKernel((void*)tl::k_vc_cg, NBc, kT, args, 0, 0));
    TL_CUDA(cudaEventRecord(e1, 0));
    TL_CUDA(cudaEventSynchronize(e1));
    TL_CUDA(cudaEventElapsedTime(&g_vc_last_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    tl::SolveInfoDev hinfo{};
    TL_CUDA(cudaMemcpy(&hinfo, dinfo, sizeof(hinfo), cudaMemcpyDeviceToHost));
    info->iterations = hinfo.iterations;
    info->status = hinfo.status;
    info->bnorm = hinfo.bnorm;
    info->rnorm = hinfo.rnorm;
    info->true_resid = hinfo.true_resid;
    *passes = pit;
    pass_iters[pit - 1] = hinfo.iterations;
    pass_ms[pit - 1] = g_vc_last_ms;
    if (hinfo.status != 0) break;                 // the caller maps the CG outcome
    if (linear) break;                            // one pass: linear problem / tl_vc_step_region_host
    // relative increment (fem.py:346-348), damped lag update (fem.py:350-354)
    tl::k_vc_inc<<<kNB, kT>>>(n, x, dTl, cpart);
    TL_CUDA(cudaGetLastError());
    double hp[2 * kNB];
    TL_CUDA(cudaMemcpy(hp, cpart, sizeof(hp), cudaMemcpyDeviceToHost));
    double dd = 0.0, xx = 0.0;
    for (int k = 0; k < kNB; ++k) { dd += hp[2 * k]; xx += hp[2 * k + 1]; }
    inc = sqrt(dd) / std::max(sqrt(xx), 1e-300);
    *inc_out = inc;
    if (inc < picard_tol || pit == picard_max) break;
    if (inc >= 0.9 * prev_inc) theta = std::max(0.25, 0.5 * theta);
    prev_inc = inc;
    tl::k_vc_lag<<<kNB, kT>>>(n, theta, x, dTl);
    TL_CUDA(cudaGetLastError());
    }
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(x_out, x, sizeof(double) * n));
    return TL_OK;
}

static int transmission_impl(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                             const double* local_values, double jump, const double* kg_T, const double* kg_v,
                             int32_t nkg, const double* kl_T, const double* kl_v, int32_t nkl, double* load_out);

// Per-device scratch buffers reused across calls of the interface helpers (grown on demand,
// never shrunk); the caller holds g_scratch_mu for the whole call.
struct Scratch {
    void* p = nullptr;
    size_t cap = 0;
};
static Scratch g_scratch[64][4];

static int scratch(int slot, size_t bytes, void** out) {
    int dev = 0;
    TL_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(TL_E_INVALID, "device ordinal out of range");
    Scratch& sc = g_scratch[dev][slot];
    if (bytes > sc.cap) {
        if (sc.p) cudaFree(sc.p);
        sc.p = nullptr;
        sc.cap = 0;
        TL_CUDA(cudaMalloc(&sc.p, bytes));
        sc.cap = bytes;
    }
    *out = sc.p;
    return TL_OK;
}

int32_t tl_overlap_feedback_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                                 const double* local_new, const double* local_old, double dt,
                                 const tl_vc_material* mat_global, const tl_vc_material* mat_local,
                                 const tl_gaussian* src, double* load_out) {
    if (!global_grid || !local_grid || !local_new || !local_old || !mat_global || !mat_local || !load_out)
        return fail(TL_E_INVALID, "null argument");
    if (!(dt > 0.0)) return fail(TL_E_INVALID, "time step must be positive");
    tl::Grid G{}, L{};
    if (int rc = make_grid(*global_grid, tl::kBottom, G, true)) return rc;
    if (int rc = make_grid(*local_grid, tl::kGamma, L, true)) return rc;
    if (tl::grid_is_2d(G) != tl::grid_is_2d(L)) return fail(TL_E_INVALID, "grids of different dimension");
    const int ng = 2 * (mat_global->nk + mat_global->nc), nl = 2 * (mat_local->nk + mat_local->nc);
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    const size_t pl = ((size_t)L.n + 31) / 32 * 32, pg = ((size_t)G.n + 31) / 32 * 32;
    void* dbl = nullptr;
    int rc = 0;
    if ((rc = scratch(3, sizeof(double) * (2 * pl + pg + ng + nl), &dbl))) return rc;
    double* dn = static_cast<double*>(dbl);
    double* dold = dn + pl;
    double* dload = dold + pl;
    double* tabs = dload + pg;
    TL_CUDA(copy_in(dn, local_new, sizeof(double) * L.n));
    TL_CUDA(copy_in(dold, local_old, sizeof(double) * L.n));
    auto upload = [&](const tl_vc_material* m, double* at, tl::VcMat& M) -> int {
        TL_CUDA(cudaMemcpy(at, m->k_T, sizeof(double) * m->nk, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(at + m->nk, m->k_v, sizeof(double) * m->nk, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(at + 2 * m->nk, m->c_T, sizeof(double) * m->nc, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(at + 2 * m->nk + m->nc, m->c_v, sizeof(double) * m->nc, cudaMemcpyHostToDevice));
        M = tl::VcMat{at, at + m->nk, at + 2 * m->nk, at + 2 * m->nk + m->nc, m->nk, m->nc,
                      m->rho, m->chi, m->S, m->T_melt, m->latent};
        return TL_OK;
    };
    tl::VcMat Mg{}, Ml{};
    if ((rc = upload(mat_global, tabs, Mg)) || (rc = upload(mat_local, tabs + ng, Ml))) return rc;
    tl::Gauss S{};
    if (src && src->on) {
        S.peak = src->peak; S.radius = src->radius; S.depth = src->depth;
        for (int a = 0; a < 3; ++a) S.center[a] = src->center[a];
        S.on = 1;
    }
    if (tl::grid_is_2d(G)) tl::k_overlap_feedback2<<<296, 256>>>(G, L, dn, dold, dt, Mg, Ml, S, dload);
    else tl::k_overlap_feedback<<<296, 256>>>(G, L, dn, dold, dt, Mg, Ml, S, dload);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(load_out, dload, sizeof(double) * G.n));
    return TL_OK;
}

int32_t tl_transmission_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                             const double* local_values, double jump, double* load_out) {
    return transmission_impl(global_grid, local_grid, local_values, jump, nullptr, nullptr, 0, nullptr, nullptr, 0,
                             load_out);
}

int32_t tl_transmission_tables_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                                    const double* local_values, const double* kg_T, const double* kg_v, int32_t nkg,
                                    const double* kl_T, const double* kl_v, int32_t nkl, double* load_out) {
    if (!kg_T || !kg_v || !kl_T || !kl_v || nkg < 2 || nkl < 2) return fail(TL_E_INVALID, "bad conductivity tables");
    return transmission_impl(global_grid, local_grid, local_values, 0.0, kg_T, kg_v, nkg, kl_T, kl_v, nkl, load_out);
}

static int transmission_impl(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                             const double* local_values, double jump, const double* kg_T, const double* kg_v,
                             int32_t nkg, const double* kl_T, const double* kl_v, int32_t nkl, double* load_out) {
    if (!global_grid || !local_grid || !local_values || !load_out) return fail(TL_E_INVALID, "null argument");
    tl::Grid G{}, L{};
    if (int rc = make_grid(*global_grid, tl::kBottom, G, true)) return rc;
    if (int rc = make_grid(*local_grid, tl::kGamma, L, true)) return rc;
    const bool two_d = tl::grid_is_2d(G);
    if (two_d != tl::grid_is_2d(L)) return fail(TL_E_INVALID, "grids of different dimension");
    // 3D: facets (triangles), 3 points x 4 pairs each; 2D: edges, 2 points x 3 pairs each
    const long long nf = two_d ? (long long)L.nc[0] + 2ll * L.nc[1]
                               : 2ll * ((long long)L.nc[1] * L.nc[2] * 2 + (long long)L.nc[0] * L.nc[2] * 2 +
                                        (long long)L.nc[0] * L.nc[1]);
    const long long ne = two_d ? 6 * nf : 12 * nf;
    if (ne >= (1ll << 31)) return fail(TL_E_INVALID, "interface too large");
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    const size_t pl = ((size_t)L.n + 31) / 32 * 32, pe = ((size_t)ne + 31) / 32 * 32, pg = ((size_t)G.n + 31) / 32 * 32;
    const size_t pt = ((size_t)2 * (nkg + nkl) + 31) / 32 * 32;
    void *dbl = nullptr, *ints = nullptr;
    int rc = 0;
    if ((rc = scratch(0, sizeof(double) * (pl + pe + pg + pt), &dbl)) || (rc = scratch(1, sizeof(int) * 4 * pe, &ints)))
        return rc;
    double* dT = static_cast<double*>(dbl);
    double* dvals = dT + pl;
    double* dload = dvals + pe;
    int* keys = static_cast<int*>(ints);
    int* keys2 = keys + pe;
    int* idx = keys2 + pe;
    int* idx2 = idx + pe;
    TL_CUDA(copy_in(dT, local_values, sizeof(double) * L.n));
    TL_CUDA(cudaMemset(dload, 0, sizeof(double) * G.n));
    double* dtab = dload + pg;
    tl::KTab kg{nullptr, nullptr, 0}, kl{nullptr, nullptr, 0};
    if (nkg > 0) {
        TL_CUDA(cudaMemcpy(dtab, kg_T, sizeof(double) * nkg, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(dtab + nkg, kg_v, sizeof(double) * nkg, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(dtab + 2 * nkg, kl_T, sizeof(double) * nkl, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(dtab + 2 * nkg + nkl, kl_v, sizeof(double) * nkl, cudaMemcpyHostToDevice));
        kg = tl::KTab{dtab, dtab + nkg, nkg};
        kl = tl::KTab{dtab + 2 * nkg, dtab + 2 * nkg + nkl, nkl};
    }
    if (two_d) tl::k_trans_entries2<<<296, 256>>>(G, L, dT, jump, kg, kl, (int)nf, keys, idx, dvals);
    else tl::k_trans_entries<<<296, 256>>>(G, L, dT, jump, kg, kl, (int)nf, keys, idx, dvals);
    TL_CUDA(cudaGetLastError());
    int bits = 1;
    while ((1ll << bits) < G.n) ++bits;
    size_t tmp_bytes = 0;
    TL_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, idx, idx2, (int)ne, 0, bits));
    void* tmp = nullptr;
    if ((rc = scratch(2, tmp_bytes + 256, &tmp))) return rc;
    TL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, idx, idx2, (int)ne, 0, bits));
    tl::k_trans_segsum<<<296, 256>>>(keys2, idx2, dvals, (int)ne, dload);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(load_out, dload, sizeof(double) * G.n));
    return TL_OK;
}

int32_t tl_mass_norms_host(const tl_grid_desc* grid, const double* a, const double* b, double* out) {
    if (!grid || !a || !out) return fail(TL_E_INVALID, "null argument");
    tl::Grid L{};
    if (int rc = make_grid(*grid, tl::kGamma, L, true)) return rc;
    constexpr int kNB = 296;
    double *da, *db = nullptr, *dpart;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)L.n, 8, (void**)&da}, {b ? (size_t)L.n : 0, 8, (void**)&db},
                                 {2 * (size_t)kNB, 8, (void**)&dpart}}))
        return rc;
    if (!b) db = nullptr;
    TL_CUDA(copy_in(da, a, sizeof(double) * L.n));
    if (b) TL_CUDA(copy_in(db, b, sizeof(double) * L.n));
    if (tl::grid_is_2d(L)) tl::k_mass_norms2<<<kNB, 256>>>(L, da, db, dpart);
    else tl::k_mass_norms<<<kNB, 256>>>(L, da, db, dpart);
    TL_CUDA(cudaGetLastError());
    double part[2 * kNB];
    TL_CUDA(cudaMemcpy(part, dpart, sizeof(part), cudaMemcpyDeviceToHost));
    out[0] = out[1] = 0.0;
    for (int k = 0; k < kNB; ++k) { out[0] += part[2 * k]; out[1] += part[2 * k + 1]; }
    return TL_OK;
}

int32_t tl_mass_norms_split_host(const tl_grid_desc* grid, const double* a, const double* b, const double* box_lo,
                                 const double* box_hi, double* out) {
    if (!grid || !a || !b || !box_lo || !box_hi || !out) return fail(TL_E_INVALID, "null argument");
    tl::Grid L{};
    if (int rc = make_grid(*grid, tl::kBottom, L, true)) return rc;
    constexpr int kNB = 296;
    double *da, *db, *dpart;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)L.n, 8, (void**)&da}, {(size_t)L.n, 8, (void**)&db},
                                 {2 * (size_t)kNB, 8, (void**)&dpart}}))
        return rc;
    TL_CUDA(copy_in(da, a, sizeof(double) * L.n));
    TL_CUDA(copy_in(db, b, sizeof(double) * L.n));
    if (tl::grid_is_2d(L)) tl::k_mass_norms_split2<<<kNB, 256>>>(L, da, db, box_lo[0], box_lo[1], box_hi[0], box_hi[1], dpart);
    else
    tl::k_mass_norms_split<<<kNB, 256>>>(L, da, db, box_lo[0], box_lo[1], box_lo[2], box_hi[0], box_hi[1],
                                         box_hi[2], dpart);
    TL_CUDA(cudaGetLastError());
    double part[2 * kNB];
    TL_CUDA(cudaMemcpy(part, dpart, sizeof(part), cudaMemcpyDeviceToHost));
    out[0] = out[1] = 0.0;
    for (int k = 0; k < kNB; ++k) { out[0] += part[2 * k]; out[1] += part[2 * k + 1]; }
    return TL_OK;
}

int32_t tl_error_l2_host(const tl_grid_desc* ref_grid, const double* ref_values, const tl_grid_desc* grid,
                         const double* values, double* out) {
    if (!ref_grid || !ref_values || !grid || !values || !out) return fail(TL_E_INVALID, "null argument");
    tl::Grid G{}, L{};
    if (int rc = make_grid(*ref_grid, tl::kBottom, G, true)) return rc;
    if (int rc = make_grid(*grid, tl::kGamma, L, true)) return rc;
    if (tl::grid_is_2d(G) != tl::grid_is_2d(L)) return fail(TL_E_INVALID, "grids of different dimension");
    constexpr int kNB = 296;
    double *dref, *dv, *dri, *dpart;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)G.n, 8, (void**)&dref}, {(size_t)L.n, 8, (void**)&dv},
                                 {(size_t)L.n, 8, (void**)&dri}, {2 * (size_t)kNB, 8, (void**)&dpart}}))
        return rc;
    TL_CUDA(copy_in(dref, ref_values, sizeof(double) * G.n));
    TL_CUDA(copy_in(dv, values, sizeof(double) * L.n));
    if (tl::grid_is_2d(G)) {
        tl::k_interp2<<<296, 256>>>(G, L, dref, dri, 0);
        tl::k_mass_norms2<<<kNB, 256>>>(L, dv, dri, dpart);
    } else {
    tl::k_interp<<<592, 256>>>(G, dref, L, 0, dri, nullptr);     // reference on the grid's nodes
    tl::k_mass_norms<<<kNB, 256>>>(L, dv, dri, dpart);
    }
    TL_CUDA(cudaGetLastError());
    double part[2 * kNB];
    TL_CUDA(cudaMemcpy(part, dpart, sizeof(part), cudaMemcpyDeviceToHost));
    out[0] = out[1] = 0.0;
    for (int k = 0; k < kNB; ++k) { out[0] += part[2 * k]; out[1] += part[2 * k + 1]; }
    return TL_OK;
}

int32_t tl_interpolate_points_host(const tl_grid_desc* global_grid, const double* values,
                                   const double* points, int64_t npoints, double* out) {
    if (!global_grid || !values || !points || !out || npoints < 0) return fail(TL_E_INVALID, "bad argument");
    tl::Grid G{};
    if (int rc = make_grid(*global_grid, tl::kBottom, G, true)) return rc;
    const int pd = tl::grid_is_2d(G) ? 2 : 3;          // doubles per point
    double *dv, *dp, *dout;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)G.n, 8, (void**)&dv}, {pd * (size_t)npoints, 8, (void**)&dp},
                                 {(size_t)npoints, 8, (void**)&dout}}))
        return rc;
    TL_CUDA(copy_in(dv, values, sizeof(double) * G.n));
    TL_CUDA(cudaMemcpy(dp, points, sizeof(double) * pd * npoints, cudaMemcpyHostToDevice));
    if (npoints > 0 && pd == 2) tl::k_interp_pts2<<<296, 256>>>(G, dv, dp, (int)npoints, dout);
    else
    if (npoints > 0) tl::k_interp_pts<<<296, 256>>>(G, dv, dp, npoints, dout);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemcpy(out, dout, sizeof(double) * npoints, cudaMemcpyDeviceToHost));
    return TL_OK;
}

int32_t tl_deposit_host(const tl_grid_desc* grid, const double* points, const double* power,
                        int32_t count, double* load_out) {
    if (!grid || !load_out || count < 0) return fail(TL_E_INVALID, "bad argument");
    if (count * 4 > tl::kDepMax) return fail(TL_E_INVALID, "too many deposit samples per call");
    tl::Grid G{};
    if (int rc = make_grid(*grid, tl::kBottom, G)) return rc;
    double *dl, *dp, *dw;
    int *prev, *prevn;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{(size_t)G.n, 8, (void**)&dl}, {3 * (size_t)count, 8, (void**)&dp},
                                 {(size_t)count, 8, (void**)&dw}, {(size_t)tl::kDepMax, 4, (void**)&prev},
                                 {1, 4, (void**)&prevn}}))
        return rc;
    TL_CUDA(cudaMemset(dl, 0, sizeof(double) * G.n));
    TL_CUDA(cudaMemset(prevn, 0, sizeof(int)));
    if (count) {
        TL_CUDA(cudaMemcpy(dp, points, sizeof(double) * 3 * count, cudaMemcpyHostToDevice));
        TL_CUDA(cudaMemcpy(dw, power, sizeof(double) * count, cudaMemcpyHostToDevice));
    }
    tl::k_deposit<<<1, 1024>>>(G, dp, dw, count, dl, prev, prevn, 0, G.n);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(load_out, dl, sizeof(double) * G.n));
    return TL_OK;
}

// ---- device vectors for callers that keep step-level fields on the device --------------
int32_t tl_dev_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return fail(TL_E_INVALID, "bad argument");
    *out = nullptr;
    TL_CUDA(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 16)));
    return TL_OK;
}

int32_t tl_dev_free(void* p) {
    if (p) TL_CUDA(cudaFree(p));
    return TL_OK;
}

int32_t tl_dev_copy(void* dst, const void* src, int64_t bytes) {
    if (!dst || !src || bytes < 0) return fail(TL_E_INVALID, "bad argument");
    const bool din = on_device(src), dout = on_device(dst);
    if (!din && dout) g_h2d_bytes += bytes;
    if (din && !dout) g_d2h_bytes += bytes;
    TL_CUDA(cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDefault));
    if (dout) TL_CUDA(cudaStreamSynchronize(nullptr));
    return TL_OK;
}

int32_t tl_host_traffic(int64_t* h2d_bytes, int64_t* d2h_bytes, int32_t reset) {
    if (h2d_bytes) *h2d_bytes = g_h2d_bytes.load();
    if (d2h_bytes) *d2h_bytes = g_d2h_bytes.load();
    if (reset) { g_h2d_bytes = 0; g_d2h_bytes = 0; }
    return TL_OK;
}

// y = a x + y over n doubles (host or device operands; the sum of interface loads)
int32_t tl_axpy_host(int64_t n, double a, const double* x, double* y) {
    if (!x || !y || n < 0 || n >= (1ll << 31)) return fail(TL_E_INVALID, "bad argument");
    const bool xd = on_device(x), yd = on_device(y);
    double *dx = const_cast<double*>(x), *dy = y;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    double *sx = nullptr, *sy = nullptr;
    if (int rc = scratch_arrays({{xd ? 0 : (size_t)n, 8, (void**)&sx}, {yd ? 0 : (size_t)n, 8, (void**)&sy}})) return rc;
    if (!xd) { TL_CUDA(copy_in(sx, x, sizeof(double) * n)); dx = sx; }
    if (!yd) { TL_CUDA(copy_in(sy, y, sizeof(double) * n)); dy = sy; }
    tl::k_axpy<<<296, 256>>>((int)n, a, dx, dy);
    TL_CUDA(cudaGetLastError());
    if (!yd) TL_CUDA(copy_out(y, dy, sizeof(double) * n));
    else TL_CUDA(cudaStreamSynchronize(nullptr));
    return TL_OK;
}

// The global field's P1 interpolant at listed nodes of a target lattice (the trace on the
// interface nodes, twolevel.py:130-142): the values k_interp writes at those nodes.
int32_t tl_interpolate_nodes_host(const tl_grid_desc* global_grid, const double* values, const tl_grid_desc* target,
                                  const int32_t* nodes, int64_t n, double* out) {
    if (!global_grid || !values || !target || !out || n < 0 || (n > 0 && !nodes)) return fail(TL_E_INVALID, "bad argument");
    tl::Grid G{}, L{};
    if (int rc = make_grid(*global_grid, tl::kBottom, G, true)) return rc;
    if (int rc = make_grid(*target, tl::kGamma, L, true)) return rc;
    if (tl::grid_is_2d(G) != tl::grid_is_2d(L)) return fail(TL_E_INVALID, "grids of different dimension");
    if (n == 0) return TL_OK;
    const bool vd = on_device(values);
    double *dv = const_cast<double*>(values), *sv = nullptr, *dout = nullptr;
    int* didx = nullptr;
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    if (int rc = scratch_arrays({{vd ? 0 : (size_t)G.n, 8, (void**)&sv}, {(size_t)n, 8, (void**)&dout},
                                 {(size_t)n, 4, (void**)&didx}}))
        return rc;
    if (!vd) { TL_CUDA(copy_in(sv, values, sizeof(double) * G.n)); dv = sv; }
    TL_CUDA(copy_in(didx, nodes, sizeof(int) * (size_t)n));
    if (tl::grid_is_2d(G)) tl::k_interp_nodes2<<<296, 256>>>(G, L, dv, didx, (int)n, dout);
    else tl::k_interp_nodes<<<296, 256>>>(G, dv, L, didx, (int)n, dout);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(copy_out(out, dout, sizeof(double) * (size_t)n));
    return TL_OK;
}

// ------------------------------------------------------------------------------------
// Device-resident run.
// ------------------------------------------------------------------------------------
int32_t tl_run_create(const tl_run_desc* desc, tl_run** out) {
    if (!desc || !out) return fail(TL_E_INVALID, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= desc->device) return fail(TL_E_NODEVICE, "no CUDA device");
    TL_CUDA(cudaSetDevice(desc->device));
    int coop = 0;
    TL_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, desc->device));
    if (!coop) return fail(TL_E_NODEVICE, "device lacks cooperative launch");
    tl_run* R = new tl_run();
    R->device = desc->device;
    R->desc = *desc;
    int rc = 0;
    if ((rc = device_sms(R->device, R->sms)) || (rc = make_grid(desc->global_grid, tl::kBottom, R->G)) ||
        (rc = make_grid(desc->local_grid, tl::kGamma, R->L))) {
        delete R;
        return rc;
    }
    if (gauss_smem(R->L) > 200 * 1024) { delete R; return fail(TL_E_INVALID, "local grid too long"); }
    TL_CUDA(cudaStreamCreateWithFlags(&R->stream, cudaStreamNonBlocking));
    const int ng = R->G.n, nl = R->L.n;
    const size_t gnxy = (size_t)R->G.NX * R->G.NY;
    if (desc->external_planes < 0 || desc->external_planes > R->G.NZ) {
        delete R;
        return fail(TL_E_INVALID, "external_planes out of range");
    }
    if (desc->external_planes > 0) {
        // the global field comes from the z-slab solve: keep only its top planes (the
        // local box's P1 support) and no global solver workspace
        R->external_global = true;
        R->ext_k0 = R->G.NZ - desc->external_planes;
        if ((rc = dalloc(&R->Tg_store, gnxy * desc->external_planes))) { tl_run_destroy(R); return rc; }
        R->Tg = R->Tg_store - (ptrdiff_t)((size_t)R->ext_k0 * gnxy);
    } else if ((rc = dalloc(&R->Tg, ng)) || (rc = dalloc(&R->bg, ng)) || (rc = dalloc(&R->rg, ng)) ||
               (rc = dalloc(&R->pg0, ng)) || (rc = dalloc(&R->pg1, ng)) || (rc = dalloc(&R->qg, ng)) ||
               (rc = dalloc(&R->loadg, ng))) {
        tl_run_destroy(R);
        return rc;
    }
    const int nxg = R->external_global ? nl : std::max(ng, nl);
    if ((rc = dalloc(&R->Tl, nl)) || (rc = dalloc(&R->bl, nl)) ||
        (rc = dalloc(&R->rl, nl)) || (rc = dalloc(&R->pl0, nl)) || (rc = dalloc(&R->pl1, nl)) ||
        (rc = dalloc(&R->ql, nl)) || (rc = dalloc(&R->tr_old, nl)) || (rc = dalloc(&R->tr_pred, nl)) ||
        (rc = dalloc(&R->Tl_before, nl)) || (rc = dalloc(&R->part, tl::kPartLen)) ||
        (rc = dalloc(&R->dep_prev, tl::kDepMax)) || (rc = dalloc(&R->dep_prev_n, 1)) ||
        (rc = dalloc(&R->melt, 4)) || (rc = dalloc(&R->melt_part, 2 * 1184)) ||
        (rc = dalloc(&R->xg, 4 * (size_t)nxg)) || (rc = dalloc(&R->d_specs, 64))) {
        tl_run_destroy(R);
        return rc;
    }
    R->specs_cap = 64;
    if (R->loadg) TL_CUDA(cudaMemsetAsync(R->loadg, 0, sizeof(double) * ng, R->stream));
    TL_CUDA(cudaMemsetAsync(R->dep_prev_n, 0, sizeof(int), R->stream));
    TL_CUDA(cudaMemsetAsync(R->tr_old, 0, sizeof(double) * nl, R->stream));
    TL_CUDA(cudaMemsetAsync(R->tr_pred, 0, sizeof(double) * nl, R->stream));
    TL_CUDA(cudaMallocHost((void**)&R->melt_host, 4 * sizeof(double)));
    *out = R;
    return TL_OK;
}

int32_t tl_run_destroy(tl_run* R) {
    if (!R) return TL_OK;
    cudaSetDevice(R->device);
    if (R->stream) cudaStreamSynchronize(R->stream);
    if (R->external_global) R->Tg = R->Tg_store;
    double* bufs[] = {R->Tg, R->bg, R->rg, R->pg0, R->pg1, R->qg, R->loadg, R->Tl, R->bl, R->rl, R->pl0,
                      R->pl1, R->ql, R->tr_old, R->tr_pred, R->Tl_before, R->part, R->dep_pts,
                      R->dep_pow, R->melt, R->melt_part, R->flush, R->xg, R->gload};
    for (double* b : bufs)
        if (b) cudaFree(b);
    if (R->dep_prev) cudaFree(R->dep_prev);
    if (R->dep_prev_n) cudaFree(R->dep_prev_n);
    if (R->info) cudaFree(R->info);
    if (R->d_specs) cudaFree(R->d_specs);
    if (R->d_srcs) cudaFree(R->d_srcs);
    if (R->gather_buf) cudaFree(R->gather_buf);
    if (R->batch_dev) cudaFree(R->batch_dev);
    if (R->batch_ctr) cudaFree(R->batch_ctr);
    if (R->snap_g) cudaFree(R->snap_g);
    for (cudaEvent_t e : R->ev) cudaEventDestroy(e);
    for (double* b : R->snap_l) cudaFree(b);
    if (R->melt_host) cudaFreeHost(R->melt_host);
    R->cache_g.release();
    R->cache_l.release();
    for (int k = 0; k < 4; ++k) {
        if (R->stage[k]) cudaFree(R->stage[k]);
        if (R->stage_ready[k]) cudaEventDestroy(R->stage_ready[k]);
        if (R->stage_done[k]) cudaEventDestroy(R->stage_done[k]);
    }
    if (R->copy_stream) {
        cudaStreamSynchronize(R->copy_stream);
        cudaStreamDestroy(R->copy_stream);
    }
    if (R->stream) cudaStreamDestroy(R->stream);
    delete R;
    return TL_OK;
}

static int run_interp_local(tl_run* R, int mode, double* out_all, double* out_gamma) {
    tl::k_interp<<<4 * R->sms, 256, 0, R->stream>>>(R->G, R->Tg, R->L, mode, out_all, out_gamma);
    ++R->launches;
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

int32_t tl_run_initial(tl_run* R, double T0) {
    if (!R) return fail(TL_E_INVALID, "null run");
    TL_CUDA(cudaSetDevice(R->device));
    for (int a = 0; a < 3; ++a) R->L.off[a] = R->desc.local_grid.offset[a];   // initial placement
    const size_t gnxy = (size_t)R->G.NX * R->G.NY;
    tl::k_fill<<<4 * R->sms, 256, 0, R->stream>>>(R->Tg + R->ext_k0 * gnxy, (int)((size_t)R->G.n - R->ext_k0 * gnxy),
                                                  T0);
    ++R->launches;
    TL_CUDA(cudaGetLastError());
    return run_interp_local(R, 0, R->Tl, R->tr_old);
}

int32_t tl_run_set_global(tl_run* R, const double* Tg_host, int64_t n) {
    if (!R || !Tg_host || n != R->G.n) return fail(TL_E_INVALID, "global field size mismatch");
    if (R->external_global) return fail(TL_E_INVALID, "external-global run: use tl_run_put_global_planes");
    TL_CUDA(cudaSetDevice(R->device));
    for (int a = 0; a < 3; ++a) R->L.off[a] = R->desc.local_grid.offset[a];   // initial placement
    TL_CUDA(cudaMemcpyAsync(R->Tg, Tg_host, sizeof(double) * n, cudaMemcpyHostToDevice, R->stream));
    return run_interp_local(R, 0, R->Tl, R->tr_old);
}

static int ensure_info(tl_run* R, int extra) {
    if (R->info_n + extra <= R->info_cap) return TL_OK;
    int cap = R->info_cap ? R->info_cap : 1024;
    while (cap < R->info_n + extra) cap *= 2;
    tl::SolveInfoDev* ni = nullptr;
    if (int rc = dalloc(&ni, cap)) return rc;
    if (R->info) {
        TL_CUDA(cudaMemcpyAsync(ni, R->info, sizeof(tl::SolveInfoDev) * R->info_n, cudaMemcpyDeviceToDevice, R->stream));
        TL_CUDA(cudaStreamSynchronize(R->stream));
        cudaFree(R->info);
    }
    R->info = ni;
    R->info_cap = cap;
    return TL_OK;
}

static void base_params(tl_run* R, tl::PcgParams& P, bool local, double dt) {
    P.g = local ? R->L : R->G;
    set_coeffs(P, R->desc.kappa, local ? R->desc.rho_c_local : R->desc.rho_c_global, dt);
    P.rtol = R->desc.rtol;
    long long mi = (long long)R->desc.maxiter_factor * P.g.n;
    P.maxiter = mi > 2000000000ll ? 2000000000 : (int)mi;
    P.part = R->part;
    if (local) {
        P.b = R->bl; P.r = R->rl; P.p0 = R->pl0; P.p1 = R->pl1; P.q = R->ql;
    } else {
        P.b = R->bg; P.r = R->rg; P.p0 = R->pg0; P.p1 = R->pg1; P.q = R->qg;
    }
}

static int ensure_snapshots(tl_run* R, int nl) {
    if (!R->snap_g)
        if (int rc = dalloc(&R->snap_g, R->G.n)) return rc;
    while ((int)R->snap_l.size() < nl) {
        double* b = nullptr;
        if (int rc = dalloc(&b, R->L.n)) return rc;
        R->snap_l.push_back(b);
    }
    return TL_OK;
}

// True when every solve of the local grid takes the streaming path (no resident kernel
// fits it, with or without Gaussian tables).
static bool local_streams(tl_run* R) {
    if (force_streaming()) return split_minb() != 0;
    if (split_minb() == 0) return false;
    BrickPlan bp;
    if (cg_fits(R->L, true, R->sms, bp) || cg_fits(R->L, false, R->sms, bp)) return false;
    return !plan_bricks(R->L, true, R->sms, 200 * 1024, false).ok && !plan_bricks(R->L, false, R->sms, 200 * 1024, false).ok;
}

// Streaming local grid: the Gaussian loads of all ns solves of a macro step by ONE
// k_gauss_loads launch, dense over the box where the term can change the RHS (bitwise the
// RHS of the per-solve k_gauss_load; tl_resident_cg.cuh), read by k_s_rhs through
// PcgParams::bload / bbox.  Replaces a full-grid pass (T read, load written) per solve and
// the load read of every RHS.
static int stream_gauss_loads(tl_run* R, const tl_macro_plan& mp, const tl_micro_plan* micro, int ns) {
    if (R->specs_cap < ns + 1) {
        if (R->d_specs) cudaFree(R->d_specs);
        R->d_specs = nullptr;
        if (int rc = dalloc(&R->d_specs, ns + 1)) return rc;
        R->specs_cap = ns + 1;
    }
    if (R->gload_cap < ns) {
        if (R->gload) cudaFree(R->gload);
        if (R->d_srcs) cudaFree(R->d_srcs);
        R->gload = nullptr;
        R->d_srcs = nullptr;
        if (int rc = dalloc(&R->gload, (size_t)ns * R->L.n)) return rc;
        if (int rc = dalloc(&R->d_srcs, ns)) return rc;
        R->gload_cap = ns;
    }
    R->h_specs.assign(ns, tl::SolveSpec{});
    R->h_srcs.assign(ns, tl::Gauss{});
    const double V = R->L.h[0] * R->L.h[1] * R->L.h[2];
    bool any = false;
    for (int e = 0; e < ns; ++e) {
        const tl_micro_plan& up = micro[mp.micro_offset + e];
        tl::SolveSpec& sp = R->h_specs[e];
        sp.mbase = (R->desc.rho_c_local / up.dt) * V / 24.0;
        sp.src.peak = R->desc.beam_peak;
        sp.src.radius = R->desc.beam_radius;
        sp.src.depth = R->desc.beam_depth;
        for (int a = 0; a < 3; ++a) sp.src.center[a] = up.center[a];
        sp.src.on = up.source_on ? 1 : 0;
        R->h_srcs[e] = sp.src;
        any = any || sp.src.on;
    }
    if (!any) return TL_OK;
    TL_CUDA(cudaMemcpyAsync(R->d_specs + 1, R->h_specs.data(), sizeof(tl::SolveSpec) * ns, cudaMemcpyHostToDevice,
                            R->stream));
    TL_CUDA(cudaMemcpyAsync(R->d_srcs, R->h_srcs.data(), sizeof(tl::Gauss) * ns, cudaMemcpyHostToDevice, R->stream));
    const size_t smem = gauss_smem(R->L);
    TL_CUDA(ensure_smem_attr((const void*)tl::k_gauss_loads, smem));
    const dim3 grid((unsigned)std::max(1, (8 * R->sms + ns - 1) / ns), (unsigned)ns);
    tl::k_gauss_loads<<<grid, 256, smem, R->stream>>>(R->L, R->d_specs + 1, R->d_srcs, 0.5 * R->desc.T_buildplate,
                                                      R->gload);
    TL_CUDA(cudaGetLastError());
    ++R->launches;
    return TL_OK;
}

// Parameters of one local solve from T; boxed >= 0: its Gaussian load was precomputed as
// entry `boxed` of stream_gauss_loads.  Returns whether an in-kernel Gaussian is still needed.
static bool local_params(tl_run* R, double* T, const tl_micro_plan& mp, int boxed, tl::PcgParams& P) {
    base_params(R, P, true, mp.dt);
    P.T = T;
    P.gA = R->tr_old;
    P.gB = R->tr_pred;
    P.w = mp.w;
    P.load = nullptr;
    bool gauss = mp.source_on != 0;
    if (gauss && boxed >= 0) {
        P.bload = R->gload + (size_t)boxed * R->L.n;
        P.bbox = (R->d_specs + 1 + boxed)->box;
        gauss = false;
    }
    if (gauss) {
        P.src.peak = R->desc.beam_peak; P.src.radius = R->desc.beam_radius; P.src.depth = R->desc.beam_depth;
        for (int a = 0; a < 3; ++a) P.src.center[a] = mp.center[a];
        P.src.on = 1;
    }
    P.info = R->info + R->info_n++;
    return gauss;
}

static int local_solve(tl_run* R, double* T, const tl_micro_plan& mp, int boxed = -1) {
    tl::PcgParams P{};
    const bool gauss = local_params(R, T, mp, boxed, P);
    if (int rc = timed_begin(R, 1)) return rc;
    if (int rc = launch_solve(P, gauss, R->sms, R->xg, R->stream, &R->launches, R->d_specs, nullptr, &R->cache_l))
        return rc;
    return timed_end(R);
}

// Snapshot decimation (tl_macro_plan::record): 1 keeps every micro field; a larger value
// keeps micro field i only if bit i + 1 is set (indices >= 30 are always kept).  The
// predicted global field and the step's final local field are kept whenever record != 0.
static inline bool keep_micro(int record, int i) {
    return record == 1 || i >= 30 || ((record >> (i + 1)) & 1);
}

// All micro solves of one macro step (+ the corrector) as one k_pcg_resident_cg launch.
static int local_multi(tl_run* R, const tl_macro_plan& mp, const tl_micro_plan* micro,
                       const BrickPlan& bp) {
    const int ns = mp.n_micro + (mp.corrector ? 1 : 0);
    if (R->specs_cap < ns + 1) {
        if (R->d_specs) cudaFree(R->d_specs);
        R->d_specs = nullptr;
        if (int rc = dalloc(&R->d_specs, ns + 1)) return rc;
        R->specs_cap = ns + 1;
    }
    R->h_specs.assign(ns, tl::SolveSpec{});
    R->h_srcs.assign(ns, tl::Gauss{});
    if (R->gload_cap < ns) {
        if (R->gload) cudaFree(R->gload);
        if (R->d_srcs) cudaFree(R->d_srcs);
        R->gload = nullptr;
        R->d_srcs = nullptr;
        if (int rc = dalloc(&R->gload, (size_t)ns * R->L.n)) return rc;
        if (int rc = dalloc(&R->d_srcs, ns)) return rc;
        R->gload_cap = ns;
    }
    bool any_src = false;
    const double V = R->L.h[0] * R->L.h[1] * R->L.h[2];
    for (int e = 0; e < ns; ++e) {
        const tl_micro_plan& up = micro[mp.micro_offset + e];
        const bool corr = mp.corrector && e == mp.n_micro;
        tl::SolveSpec& sp = R->h_specs[e];
        sp.mbase = (R->desc.rho_c_local / up.dt) * V / 24.0;      // set_coeffs
        sp.w = up.w;
        sp.src.peak = R->desc.beam_peak;
        sp.src.radius = R->desc.beam_radius;
        sp.src.depth = R->desc.beam_depth;
        for (int a = 0; a < 3; ++a) sp.src.center[a] = up.center[a];
        sp.src.on = up.source_on ? 1 : 0;
        // the Gaussian is precomputed for all solves by k_gauss_loads (no in-kernel tables)
        R->h_srcs[e] = sp.src;
        sp.load = sp.src.on ? R->gload + (size_t)e * R->L.n : nullptr;
        any_src = any_src || sp.src.on;
        sp.src.on = 0;
        sp.tin = corr ? 2 : (e == 0 ? 0 : 1);
        sp.save_before = (mp.corrector && e == mp.n_micro - 1) ? 1 : 0;
        sp.tout = (e == ns - 1) ? 1 : 0;
        sp.info = R->info + R->info_n++;
        sp.snap = nullptr;
        if (mp.record) {
            if (int rc = ensure_snapshots(R, ns)) return rc;
            if (e == ns - 1 || keep_micro(mp.record, e)) sp.snap = R->snap_l[e];
        }
    }
    TL_CUDA(cudaMemcpyAsync(R->d_specs + 1, R->h_specs.data(), sizeof(tl::SolveSpec) * ns,
                            cudaMemcpyHostToDevice, R->stream));
    if (any_src) {
        TL_CUDA(cudaMemcpyAsync(R->d_srcs, R->h_srcs.data(), sizeof(tl::Gauss) * ns, cudaMemcpyHostToDevice,
                                R->stream));
        const size_t smem = gauss_smem(R->L);
        TL_CUDA(ensure_smem_attr((const void*)tl::k_gauss_loads, smem));
        // the box of each solve is ~15 % of the local grid: spread it over the whole GPU
        const dim3 grid((unsigned)std::max(1, (8 * R->sms + ns - 1) / ns), (unsigned)ns);
        tl::k_gauss_loads<<<grid, 256, smem, R->stream>>>(R->L, R->d_specs + 1, R->d_srcs,
                                                          0.5 * R->desc.T_buildplate, R->gload);
        TL_CUDA(cudaGetLastError());
        ++R->launches;
    }
    tl::PcgParams P{};
    base_params(R, P, true, micro[mp.micro_offset].dt);
    P.T = R->Tl;
    P.gA = R->tr_old;
    P.gB = R->tr_pred;
    P.load = nullptr;
    tl::ResCGParams RP{};
    fill_rescg(RP, P, R->xg, bp);
    RP.specs = R->d_specs + 1;
    RP.nspec = ns;
    if (getenv("TLGPU_NOCACHE") == nullptr)
        if (int rc = attach_cache(&R->cache_l, RP, R->L, bp)) return rc;
    const int G = bp.ng[0] * bp.ng[1] * bp.ng[2];
    if (int rc = timed_begin(R, 1, ns)) return rc;
    cudaError_t e = launch_rescg_g<false, true>(RP, bp.npt, G, bp.smem, R->stream);
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("k_pcg_resident_cg (multi) launch: ") + cudaGetErrorString(e));
    ++R->launches;
    if (RP.scache) R->cache_l.ready = true;
    return timed_end(R);
}

// One macro step's global part (twolevel.solve_global + the predicted trace) on the run's
// stream: deposit, implicit step, snapshot, trace interpolation.
static int step_global_phase(tl_run* R, const tl_macro_plan& mp) {
    // -- global predictor (twolevel.solve_global): deposit + implicit step --
    if (!R->external_global) {
    tl::k_deposit<<<1, 1024, 0, R->stream>>>(R->G, R->dep_pts + 3 * (size_t)mp.dep_offset,
                                             R->dep_pow + mp.dep_offset, mp.dep_count, R->loadg,
                                             R->dep_prev, R->dep_prev_n, 0, R->G.n);
    ++R->launches;
    TL_CUDA(cudaGetLastError());
    tl::PcgParams P{};
    base_params(R, P, false, mp.dt_global);
    P.T = R->Tg;
    P.gA = nullptr;
    P.g_const = R->desc.T_buildplate;
    P.load = R->loadg;
    P.info = R->info + R->info_n++;
    if (int rc = timed_begin(R, 0)) return rc;
    if (int rc = launch_solve(P, false, R->sms, R->xg, R->stream, &R->launches, R->d_specs, nullptr,
                              &R->cache_g))
        return rc;
    if (int rc = timed_end(R)) return rc;
    }
    if (mp.record) {
        if (int rc = ensure_snapshots(R, mp.n_micro + mp.corrector)) return rc;
        TL_CUDA(cudaMemcpyAsync(R->snap_g, R->Tg, sizeof(double) * R->G.n, cudaMemcpyDeviceToDevice, R->stream));
        R->snap_n = mp.n_micro + mp.corrector;
    }
    // -- trace of the predicted global field on gamma --
    if (int rc = run_interp_local(R, 1, nullptr, R->tr_pred)) return rc;
    return TL_OK;
}

// End of a macro step: the converged trace, then the relocation (scanpath.relocate_local).
static int step_finish_phase(tl_run* R, const tl_macro_plan& mp) {
    // converged trace at the macro instant = trace_pred
    std::swap(R->tr_old, R->tr_pred);
    if (mp.relocate) {
        for (int a = 0; a < 3; ++a) R->L.off[a] = mp.new_offset[a];
        if (int rc = run_interp_local(R, 0, R->Tl, R->tr_old)) return rc;
    }
    return TL_OK;
}

int32_t tl_run_macro_steps(tl_run* R, const tl_macro_plan* plans, int32_t nsteps,
                           const tl_micro_plan* micro, int32_t nmicro, const double* dep_points,
                           const double* dep_power, int32_t ndep) {
    if (!R || (!plans && nsteps > 0)) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    BrickPlan lbp;
    // All micro solves + the corrector of a macro step in one persistent launch when the
    // local grid fits the resident CG-CG kernel (Gaussian loads precomputed by one
    // k_gauss_loads launch, setup shared by the solves, one launch instead of 11: cfg2
    // 2.16 vs 2.21 ms per step).  TLGPU_MULTI=0: one launch per solve.
    const char* mv = getenv("TLGPU_MULTI");
    const bool multi = !(mv && mv[0] == '0') && cg_fits(R->L, false, R->sms, lbp) &&
                       !(lbp.xglob && getenv("TLGPU_NOCACHE"));
    // TLGPU_BOXLOAD=0: per-solve k_gauss_load over the whole local grid (streaming path)
    const char* bv = getenv("TLGPU_BOXLOAD");
    const bool lstream = !(bv && bv[0] == '0') && !multi && local_streams(R);

    int need = 0;
    for (int s = 0; s < nsteps; ++s) {
        const tl_macro_plan& mp = plans[s];
        if (mp.n_micro < 1 || mp.micro_offset < 0 || mp.micro_offset + mp.n_micro + mp.corrector > nmicro)
            return fail(TL_E_INVALID, "micro plan out of range");
        if (mp.dep_count < 0 || mp.dep_offset < 0 || mp.dep_offset + mp.dep_count > ndep)
            return fail(TL_E_INVALID, "deposit plan out of range");
        if (mp.dep_count * 4 > tl::kDepMax) return fail(TL_E_INVALID, "too many deposit samples in one step");
        if (mp.record && R->external_global) return fail(TL_E_INVALID, "external-global runs keep no snapshots");
        need += (R->external_global ? 0 : 1) + mp.n_micro + mp.corrector;
    }
    if (int rc = ensure_info(R, need)) return rc;
    if (ndep > R->dep_cap) {
        if (R->dep_pts) cudaFree(R->dep_pts);
        if (R->dep_pow) cudaFree(R->dep_pow);
        int rc = 0;
        if ((rc = dalloc(&R->dep_pts, 3 * (size_t)ndep)) || (rc = dalloc(&R->dep_pow, ndep))) return rc;
        R->dep_cap = ndep;
    }
    if (ndep > 0) {
        TL_CUDA(cudaMemcpyAsync(R->dep_pts, dep_points, sizeof(double) * 3 * ndep, cudaMemcpyHostToDevice, R->stream));
        TL_CUDA(cudaMemcpyAsync(R->dep_pow, dep_power, sizeof(double) * ndep, cudaMemcpyHostToDevice, R->stream));
    }
    for (int s = 0; s < nsteps; ++s) {
        const tl_macro_plan& mp = plans[s];
        if (int rc = step_global_phase(R, mp)) return rc;
        // -- micro steps (+ corrector): one persistent launch when the local grid fits --
        const bool boxed = !multi && lstream;
        if (boxed)
            if (int rc = stream_gauss_loads(R, mp, micro, mp.n_micro + (mp.corrector ? 1 : 0))) return rc;
        if (multi) {
            if (int rc = local_multi(R, mp, micro, lbp)) return rc;
        } else
        for (int i = 0; i < mp.n_micro; ++i) {
            const tl_micro_plan& up = micro[mp.micro_offset + i];
            if (i == mp.n_micro - 1 && mp.corrector) {
                tl::k_copy<<<4 * R->sms, 256, 0, R->stream>>>(R->Tl, R->Tl_before, R->L.n);
                ++R->launches;
            }
            if (int rc = local_solve(R, R->Tl, up, boxed ? i : -1)) return rc;
            if (mp.record && ((i == mp.n_micro - 1 && !mp.corrector) || keep_micro(mp.record, i)))
                TL_CUDA(cudaMemcpyAsync(R->snap_l[i], R->Tl, sizeof(double) * R->L.n, cudaMemcpyDeviceToDevice, R->stream));
        }
        if (mp.corrector && !multi) {
            // corrector: re-solve the last micro interval from before_final with trace_pred
            if (int rc = local_solve(R, R->Tl_before, micro[mp.micro_offset + mp.n_micro], boxed ? mp.n_micro : -1))
                return rc;
            std::swap(R->Tl, R->Tl_before);
            if (mp.record)
                TL_CUDA(cudaMemcpyAsync(R->snap_l[mp.n_micro], R->Tl, sizeof(double) * R->L.n, cudaMemcpyDeviceToDevice, R->stream));
        }
        if (int rc = step_finish_phase(R, mp)) return rc;
    }
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

// ---- batched runs (BASELINE config 5) ------------------------------------------------
// One macro step of a group of runs whose local grids have one shape: the global parts run
// per run, the i-th micro solve (and the corrector) of ALL runs is one batched solve
// (k_sb_rhs -> k_tb_cg -> k_sb_resid -> k_sb_final, tl_tiled.cuh).  Everything is enqueued
// on the first run's stream; the other runs' streams are ordered before and after it.
static int batched_solve(std::vector<tl::PcgParams>& Ps, tl_run* R0, int sms, cudaStream_t st, int64_t* launches) {
    const int B = (int)Ps.size();
    if (B == 0) return TL_OK;
    if (B > tl::kTBMax) return fail(TL_E_INVALID, "too many systems in one batched solve");
    tl::TPlan tp{};
    size_t smem = 0;
    if (!tiled_plan_range(Ps[0].g, sms, 0, Ps[0].g.NZ, tp, smem, B)) return fail(TL_E_INVALID, "no item plan for the batch");
    if ((long long)tp.I * B > 2000000000ll / 4) return fail(TL_E_INVALID, "batch too large");
    tp.iid.init((uint32_t)tp.I);
    // the parameter buffer belongs to the first run: ordered by its stream
    if (!R0->batch_dev) {
        TL_CUDA(cudaMalloc((void**)&R0->batch_dev, sizeof(tl::PcgParams) * tl::kTBMax));
        TL_CUDA(cudaMalloc((void**)&R0->batch_ctr, 4 * sizeof(unsigned)));
    }
    tl::PcgParams* dPs = static_cast<tl::PcgParams*>(R0->batch_dev);
    for (auto& P : Ps) {
        P.light_rhs = 1;
        P.snake = snake_enabled();
        P.prof = nullptr;
    }
    // stream-ordered after the previous batched solve's kernels; the pageable source is
    // staged before the call returns
    TL_CUDA(cudaMemcpyAsync(dPs, Ps.data(), sizeof(tl::PcgParams) * B, cudaMemcpyHostToDevice, st));
    static thread_local int occ_rhs = 0, occ_res = 0;
    if (occ_rhs == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_rhs, tl::k_sb_rhs, tl::kSTPB, 0) != cudaSuccess || occ_rhs < 1)
            occ_rhs = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_res, tl::k_sb_resid, tl::kSTPB, 0) != cudaSuccess || occ_res < 1)
            occ_res = 1;
    }
    // blocks per system: the batch fills the device together
    const int per = std::max(1, (std::min(4, occ_rhs) * sms + B - 1) / B);
    const int Gr = std::min(per, (Ps[0].g.n + tl::kSTPB - 1) / tl::kSTPB);
    const int perq = std::max(1, (std::min(4, occ_res) * sms + B - 1) / B);
    const int Gq = std::min(perq, (Ps[0].g.n + tl::kSTPB - 1) / tl::kSTPB);
    tl::k_sb_rhs<<<dim3(Gr, B), tl::kSTPB, 0, st>>>(dPs);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemsetAsync(R0->batch_ctr, 0, 4 * sizeof(unsigned), st));
    const int nodes = tp.H * Ps[0].g.NX;
    const int npt = nodes <= tp.ncw * 32 ? 1 : (nodes <= 2 * tp.ncw * 32 ? 2 : 4);
    auto kern = tp.ncw == 16 ? (npt == 1 ? tl::k_tb_cg<16, 1> : npt == 2 ? tl::k_tb_cg<16, 2> : tl::k_tb_cg<16, 4>)
                             : (npt == 1 ? tl::k_tb_cg<19, 1> : npt == 2 ? tl::k_tb_cg<19, 2> : tl::k_tb_cg<19, 4>);
    TL_CUDA(ensure_smem_attr((const void*)kern, smem));
    int Bv = B, Grv = Gr;
    unsigned* ctr = R0->batch_ctr;
    void* args[] = {&dPs, &Bv, &Grv, (void*)&tp, &ctr};
    TL_CUDA(cudaLaunchCooperativeKernel((void*)kern, sms, (tp.ncw + 1) * 32, args, smem, st));
    tl::k_sb_resid<<<dim3(Gq, B), tl::kSTPB, 0, st>>>(dPs);
    tl::k_sb_final<<<B, tl::kSTPB, 0, st>>>(dPs, Gq);
    TL_CUDA(cudaGetLastError());
    if (launches) *launches += 4;
    return TL_OK;
}

int32_t tl_runs_macro_step(tl_run** runs, int32_t nruns, const tl_macro_plan* plans,
                           const tl_micro_plan* const* micro, const int32_t* nmicro,
                           const double* const* dep_points, const double* const* dep_power, const int32_t* ndep) {
    if (!runs || nruns < 1 || !plans || !micro || !nmicro || !dep_points || !dep_power || !ndep)
        return fail(TL_E_INVALID, "null argument");
    if (nruns > tl::kTBMax) return fail(TL_E_INVALID, "at most 64 runs per batched step");
    tl_run* R0 = runs[0];
    TL_CUDA(cudaSetDevice(R0->device));
    for (int r = 0; r < nruns; ++r) {
        tl_run* R = runs[r];
        const tl_macro_plan& mp = plans[r];
        if (!R || R->device != R0->device) return fail(TL_E_INVALID, "batched runs must share a device");
        for (int a = 0; a < 3; ++a)
            if (R->L.nc[a] != R0->L.nc[a]) return fail(TL_E_INVALID, "batched runs need local grids of one shape");
        if (R->external_global) return fail(TL_E_INVALID, "batched runs hold their own global field");
        if (mp.record) return fail(TL_E_INVALID, "batched steps keep no snapshots");
        if (mp.n_micro < 1 || mp.micro_offset < 0 || mp.micro_offset + mp.n_micro + mp.corrector > nmicro[r])
            return fail(TL_E_INVALID, "micro plan out of range");
        if (mp.dep_count < 0 || mp.dep_offset < 0 || mp.dep_offset + mp.dep_count > ndep[r])
            return fail(TL_E_INVALID, "deposit plan out of range");
        if (mp.dep_count * 4 > tl::kDepMax) return fail(TL_E_INVALID, "too many deposit samples in one step");
        if (int rc = ensure_info(R, 1 + mp.n_micro + mp.corrector)) return rc;
    }
    // one stream for the whole step: the other runs' streams first catch up with it
    cudaStream_t S = R0->stream;
    std::vector<cudaStream_t> own(nruns);
    cudaEvent_t ev;
    TL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (int r = 0; r < nruns; ++r) {
        own[r] = runs[r]->stream;
        if (r > 0) {
            TL_CUDA(cudaEventRecord(ev, own[r]));
            TL_CUDA(cudaStreamWaitEvent(S, ev, 0));
        }
        runs[r]->stream = S;
    }
    int rc = TL_OK;
    auto restore = [&]() {
        cudaEventRecord(ev, S);
        for (int r = 0; r < nruns; ++r) {
            runs[r]->stream = own[r];
            if (r > 0) cudaStreamWaitEvent(own[r], ev, 0);
        }
        cudaEventDestroy(ev);
    };
    int max_m = 0;
    for (int r = 0; r < nruns && rc == TL_OK; ++r) {
        tl_run* R = runs[r];
        const tl_macro_plan& mp = plans[r];
        if (ndep[r] > R->dep_cap) {
            if (R->dep_pts) cudaFree(R->dep_pts);
            if (R->dep_pow) cudaFree(R->dep_pow);
            R->dep_pts = nullptr; R->dep_pow = nullptr; R->dep_cap = 0;
            if ((rc = dalloc(&R->dep_pts, 3 * (size_t)ndep[r])) || (rc = dalloc(&R->dep_pow, ndep[r]))) break;
            R->dep_cap = ndep[r];
        }
        if (ndep[r] > 0) {
            cudaMemcpyAsync(R->dep_pts, dep_points[r], sizeof(double) * 3 * ndep[r], cudaMemcpyHostToDevice, S);
            cudaMemcpyAsync(R->dep_pow, dep_power[r], sizeof(double) * ndep[r], cudaMemcpyHostToDevice, S);
        }
        // global predictor: the deposit per run, the implicit steps of all runs batched below
        tl::k_deposit<<<1, 1024, 0, S>>>(R->G, R->dep_pts + 3 * (size_t)mp.dep_offset, R->dep_pow + mp.dep_offset,
                                         mp.dep_count, R->loadg, R->dep_prev, R->dep_prev_n, 0, R->G.n);
        ++R->launches;
        max_m = std::max(max_m, mp.n_micro);
    }
    std::vector<tl::PcgParams> Ps;
    bool same_global = true;
    for (int r = 1; r < nruns; ++r)
        for (int a = 0; a < 3; ++a) same_global = same_global && runs[r]->G.nc[a] == R0->G.nc[a];
    if (rc == TL_OK && same_global) {
        for (int r = 0; r < nruns; ++r) {
            tl_run* R = runs[r];
            tl::PcgParams P{};
            base_params(R, P, false, plans[r].dt_global);
            P.T = R->Tg;
            P.gA = nullptr;
            P.g_const = R->desc.T_buildplate;
            P.load = R->loadg;
            P.info = R->info + R->info_n++;
            Ps.push_back(P);
        }
        if ((rc = timed_begin(R0, 0, nruns)) == TL_OK && (rc = batched_solve(Ps, R0, R0->sms, S, &R0->launches)) == TL_OK)
            rc = timed_end(R0);
    } else if (rc == TL_OK) {
        for (int r = 0; r < nruns && rc == TL_OK; ++r) {      // global grids differ: one solve per run
            tl_run* R = runs[r];
            tl::PcgParams P{};
            base_params(R, P, false, plans[r].dt_global);
            P.T = R->Tg;
            P.gA = nullptr;
            P.g_const = R->desc.T_buildplate;
            P.load = R->loadg;
            P.info = R->info + R->info_n++;
            rc = launch_solve(P, false, R->sms, R->xg, S, &R->launches, R->d_specs, nullptr, &R->cache_g);
        }
    }
    for (int r = 0; r < nruns && rc == TL_OK; ++r) {
        tl_run* R = runs[r];
        if ((rc = run_interp_local(R, 1, nullptr, R->tr_pred))) break;        // predicted trace on gamma
        rc = stream_gauss_loads(R, plans[r], micro[r], plans[r].n_micro + (plans[r].corrector ? 1 : 0));
    }
    for (int i = 0; i < max_m && rc == TL_OK; ++i) {
        Ps.clear();
        for (int r = 0; r < nruns; ++r) {
            tl_run* R = runs[r];
            const tl_macro_plan& mp = plans[r];
            if (i >= mp.n_micro) continue;
            if (i == mp.n_micro - 1 && mp.corrector) {
                tl::k_copy<<<4 * R->sms, 256, 0, S>>>(R->Tl, R->Tl_before, R->L.n);
                ++R->launches;
            }
            tl::PcgParams P{};
            local_params(R, R->Tl, micro[r][mp.micro_offset + i], i, P);
            Ps.push_back(P);
        }
        if ((rc = timed_begin(R0, 1, (int)Ps.size())) == TL_OK &&
            (rc = batched_solve(Ps, R0, R0->sms, S, &R0->launches)) == TL_OK)
            rc = timed_end(R0);
    }
    if (rc == TL_OK) {                      // correctors: the last micro interval again, from before_final
        Ps.clear();
        for (int r = 0; r < nruns; ++r) {
            tl_run* R = runs[r];
            const tl_macro_plan& mp = plans[r];
            if (!mp.corrector) continue;
            tl::PcgParams P{};
            local_params(R, R->Tl_before, micro[r][mp.micro_offset + mp.n_micro], mp.n_micro, P);
            Ps.push_back(P);
        }
        if (!Ps.empty() && (rc = timed_begin(R0, 1, (int)Ps.size())) == TL_OK &&
            (rc = batched_solve(Ps, R0, R0->sms, S, &R0->launches)) == TL_OK)
            rc = timed_end(R0);
        for (int r = 0; r < nruns; ++r)
            if (plans[r].corrector) std::swap(runs[r]->Tl, runs[r]->Tl_before);
    }
    for (int r = 0; r < nruns && rc == TL_OK; ++r) rc = step_finish_phase(runs[r], plans[r]);
    restore();
    if (rc == TL_OK && cudaGetLastError() != cudaSuccess) rc = fail(TL_E_CUDA, "batched macro step launch failed");
    return rc;
}

int32_t tl_run_get_snapshot(tl_run* R, int32_t which, int32_t index, double* host, int64_t n) {
    if (!R || !host) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    const double* src = nullptr;
    if (which == 0 && R->snap_g && n == R->G.n) src = R->snap_g;
    if (which == 1 && index >= 0 && index < R->snap_n && n == R->L.n) src = R->snap_l[index];
    if (!src) return fail(TL_E_INVALID, "no such snapshot");
    TL_CUDA(cudaMemcpyAsync(host, src, sizeof(double) * n, cudaMemcpyDeviceToHost, R->stream));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    return TL_OK;
}

int32_t tl_run_sync(tl_run* R) {
    if (!R) return fail(TL_E_INVALID, "null run");
    TL_CUDA(cudaSetDevice(R->device));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    return TL_OK;
}

int32_t tl_run_get_field(tl_run* R, int32_t which, double* host, int64_t n) {
    if (!R || !host) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    const double* src = which == 0 ? R->Tg : (which == 1 ? R->Tl : R->tr_old);
    const int64_t want = which == 0 ? R->G.n : R->L.n;
    if (which < 0 || which > 2 || n != want) return fail(TL_E_INVALID, "field selector or size mismatch");
    if (which == 0 && R->external_global) return fail(TL_E_INVALID, "external-global run holds no global field");
    TL_CUDA(cudaMemcpyAsync(host, src, sizeof(double) * n, cudaMemcpyDeviceToHost, R->stream));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    return TL_OK;
}

int32_t tl_run_get_field_at(tl_run* R, int32_t which, const int32_t* idx, int64_t n, double* host) {
    if (!R || !host || (!idx && n > 0) || n < 0) return fail(TL_E_INVALID, "bad argument");
    TL_CUDA(cudaSetDevice(R->device));
    const double* src = which == 0 ? R->Tg : (which == 1 ? R->Tl : R->tr_old);
    if (which < 0 || which > 2) return fail(TL_E_INVALID, "field selector");
    if (which == 0 && R->external_global) return fail(TL_E_INVALID, "external-global run holds no global field");
    if (n == 0) return TL_OK;
    const size_t need = (size_t)n * (sizeof(int) + sizeof(double)) + 16;
    if (need > R->gather_cap) {
        if (R->gather_buf) cudaFree(R->gather_buf);
        R->gather_buf = nullptr;
        R->gather_cap = 0;
        TL_CUDA(cudaMalloc(&R->gather_buf, need));
        R->gather_cap = need;
    }
    double* dval = static_cast<double*>(R->gather_buf);
    int* didx = reinterpret_cast<int*>(dval + n);
    TL_CUDA(cudaMemcpyAsync(didx, idx, sizeof(int) * n, cudaMemcpyHostToDevice, R->stream));
    tl::k_gather<<<(int)std::min<int64_t>((n + 255) / 256, 4 * R->sms), 256, 0, R->stream>>>(src, didx, (int)n, dval);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemcpyAsync(host, dval, sizeof(double) * n, cudaMemcpyDeviceToHost, R->stream));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    return TL_OK;
}

int32_t tl_run_field_async(tl_run* R, int32_t which, double* host, int64_t n, int32_t slot) {
    if (!R || !host) return fail(TL_E_INVALID, "null argument");
    if (slot < 0 || slot > 3) return fail(TL_E_INVALID, "read-back slot must be 0..3");
    TL_CUDA(cudaSetDevice(R->device));
    const double* src = which == 0 ? R->Tg : (which == 1 ? R->Tl : R->tr_old);
    const int64_t want = which == 0 ? R->G.n : R->L.n;
    if (which < 0 || which > 2 || n != want) return fail(TL_E_INVALID, "field selector or size mismatch");
    if (which == 0 && R->external_global) return fail(TL_E_INVALID, "external-global run holds no global field");
    if (!R->copy_stream) TL_CUDA(cudaStreamCreateWithFlags(&R->copy_stream, cudaStreamNonBlocking));
    if (!R->stage_ready[slot]) {
        TL_CUDA(cudaEventCreateWithFlags(&R->stage_ready[slot], cudaEventDisableTiming));
        TL_CUDA(cudaEventCreateWithFlags(&R->stage_done[slot], cudaEventDisableTiming));
    }
    if (R->stage_n[slot] < (size_t)n) {
        // the previous transfer out of this slot must have finished before it is freed
        TL_CUDA(cudaEventSynchronize(R->stage_done[slot]));
        if (R->stage[slot]) cudaFree(R->stage[slot]);
        R->stage[slot] = nullptr;
        if (int rc = dalloc(&R->stage[slot], (size_t)n)) return rc;
        R->stage_n[slot] = (size_t)n;
    }
    // the staging slot may still be read by the slot's previous transfer
    TL_CUDA(cudaStreamWaitEvent(R->stream, R->stage_done[slot], 0));
    TL_CUDA(cudaMemcpyAsync(R->stage[slot], src, sizeof(double) * n, cudaMemcpyDeviceToDevice, R->stream));
    TL_CUDA(cudaEventRecord(R->stage_ready[slot], R->stream));
    TL_CUDA(cudaStreamWaitEvent(R->copy_stream, R->stage_ready[slot], 0));
    TL_CUDA(cudaMemcpyAsync(host, R->stage[slot], sizeof(double) * n, cudaMemcpyDeviceToHost, R->copy_stream));
    TL_CUDA(cudaEventRecord(R->stage_done[slot], R->copy_stream));
    return TL_OK;
}

int32_t tl_run_field_wait(tl_run* R, int32_t slot) {
    if (!R) return fail(TL_E_INVALID, "null argument");
    if (slot < 0 || slot > 3) return fail(TL_E_INVALID, "read-back slot must be 0..3");
    if (!R->stage_done[slot]) return TL_OK;
    TL_CUDA(cudaSetDevice(R->device));
    TL_CUDA(cudaEventSynchronize(R->stage_done[slot]));
    return TL_OK;
}

int32_t tl_run_take_info(tl_run* R, tl_solve_info* out, int32_t max, int32_t* count) {
    if (!R || !count) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    const int n = R->info_n < max ? R->info_n : max;
    std::vector<tl::SolveInfoDev> tmp(n > 0 ? n : 1);
    if (n > 0) TL_CUDA(cudaMemcpy(tmp.data(), R->info, sizeof(tl::SolveInfoDev) * n, cudaMemcpyDeviceToHost));
    for (int e = 0; e < n; ++e) {
        out[e].iterations = tmp[e].iterations; out[e].status = tmp[e].status; out[e].bnorm = tmp[e].bnorm;
        out[e].rnorm = tmp[e].rnorm; out[e].true_resid = tmp[e].true_resid;
    }
    if (n < R->info_n) {   // keep the remainder at the front
        TL_CUDA(cudaMemcpy(R->info, R->info + n, sizeof(tl::SolveInfoDev) * (R->info_n - n), cudaMemcpyDeviceToDevice));
    }
    R->info_n -= n;
    *count = n;
    return TL_OK;
}

int32_t tl_run_melt_summary(tl_run* R, double T_liquidus, double* out4) {
    if (!R || !out4) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    const int nb = 4 * R->sms;
    const size_t gnxy = (size_t)R->G.NX * R->G.NY;     // external mode: the stored planes
    tl::k_melt_partial<<<nb, 256, 0, R->stream>>>(R->Tg + R->ext_k0 * gnxy,
                                                  (int)((size_t)R->G.n - R->ext_k0 * gnxy), T_liquidus, R->melt_part);
    tl::k_melt_final<<<1, 32, 0, R->stream>>>(R->melt_part, nb, R->melt + 0, R->melt + 2);
    tl::k_melt_partial<<<nb, 256, 0, R->stream>>>(R->Tl, R->L.n, T_liquidus, R->melt_part);
    tl::k_melt_final<<<1, 32, 0, R->stream>>>(R->melt_part, nb, R->melt + 1, R->melt + 3);
    R->launches += 4;
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemcpyAsync(R->melt_host, R->melt, 4 * sizeof(double), cudaMemcpyDeviceToHost, R->stream));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    for (int e = 0; e < 4; ++e) out4[e] = R->melt_host[e];
    return TL_OK;
}

int32_t tl_run_stream(tl_run* R, void** stream) {
    if (!R || !stream) return fail(TL_E_INVALID, "null argument");
    *stream = (void*)R->stream;
    return TL_OK;
}

int64_t tl_run_launch_count(tl_run* R) { return R ? R->launches : -1; }

int32_t tl_debug_profile(uint64_t* out, int32_t max, int32_t* count) {
    if (!out || !count) return fail(TL_E_INVALID, "null argument");
    *count = 0;
    if (!g_prof) return TL_OK;
    std::vector<unsigned long long> h(kProfLen);
    TL_CUDA(cudaDeviceSynchronize());
    TL_CUDA(cudaMemcpy(h.data(), g_prof, kProfLen * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    // slots [0, h[127]) phase stamps, 120..122 setup stamps, 127 = stamp count; from 1024:
    // k_t_cg's per-CTA sweep stamps (tl_tiled.cuh)
    const int n = std::min(max, kProfLen);
    for (int e = 0; e < n; ++e) out[e] = h[e];
    *count = n;
    return TL_OK;
}

int32_t tl_run_set_timing(tl_run* R, int32_t on) {
    if (!R) return fail(TL_E_INVALID, "null run");
    R->timing = on != 0;
    return TL_OK;
}

int32_t tl_run_take_timing(tl_run* R, float* ms, int32_t* level, int32_t* nsolve, int32_t max,
                           int32_t* count) {
    if (!R || !count) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    TL_CUDA(cudaStreamSynchronize(R->stream));
    const int n = R->ev_n < max ? R->ev_n : max;
    for (int e = 0; e < n; ++e) {
        float t = 0.f;
        TL_CUDA(cudaEventElapsedTime(&t, R->ev[2 * e], R->ev[2 * e + 1]));
        ms[e] = t;
        level[e] = R->ev_level[e];
        if (nsolve) nsolve[e] = R->ev_nsolve[e];
    }
    // drop the pairs we returned (keep the rest in order)
    for (int e = n; e < R->ev_n; ++e) {
        std::swap(R->ev[2 * (e - n)], R->ev[2 * e]);
        std::swap(R->ev[2 * (e - n) + 1], R->ev[2 * e + 1]);
        R->ev_level[e - n] = R->ev_level[e];
        R->ev_nsolve[e - n] = R->ev_nsolve[e];
    }
    R->ev_n -= n;
    *count = n;
    return TL_OK;
}

int32_t tl_run_flush_l2(tl_run* R) {
    if (!R) return fail(TL_E_INVALID, "null run");
    TL_CUDA(cudaSetDevice(R->device));
    if (!R->flush) {
        int l2 = 0;
        TL_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, R->device));
        R->flush_n = (size_t)l2 * 2 / sizeof(double);
        if (int rc = dalloc(&R->flush, R->flush_n)) return rc;
    }
    tl::k_flush<<<4 * R->sms, 512, 0, R->stream>>>(R->flush, R->flush_n, 1.0);
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

int32_t tl_run_reanchor(tl_run* R, const double* offset) {
    if (!R || !offset) return fail(TL_E_INVALID, "null argument");
    TL_CUDA(cudaSetDevice(R->device));
    for (int a = 0; a < 3; ++a) R->L.off[a] = offset[a];
    return run_interp_local(R, 0, R->Tl, R->tr_old);
}

int32_t tl_run_put_global_planes(tl_run* R, const double* src, int32_t k0, int32_t k1) {
    if (!R || !src) return fail(TL_E_INVALID, "null argument");
    if (k0 < R->ext_k0 || k1 > R->G.NZ || k0 >= k1) return fail(TL_E_INVALID, "bad plane range");
    TL_CUDA(cudaSetDevice(R->device));
    const size_t nxy = (size_t)R->G.NX * R->G.NY;
    TL_CUDA(cudaMemcpyAsync(R->Tg + (size_t)k0 * nxy, src, sizeof(double) * nxy * (k1 - k0),
                            cudaMemcpyDeviceToDevice, R->stream));
    return TL_OK;
}

// ---- z-slab global solve (multi-GPU) ----------------------------------------------

static int slab_params(const tl_slab* s, tl::SlabParams& S, int& blocks, cudaStream_t& st) {
    if (!s || !s->x || !s->b || !s->r || !s->p0 || !s->p1 || !s->work || !s->sums)
        return fail(TL_E_INVALID, "null slab argument");
    if (s->dirichlet_kind != tl::kBottom) return fail(TL_E_INVALID, "slabs support TL_DIRICHLET_BOTTOM only");
    if (s->dt <= 0) return fail(TL_E_INVALID, "time step must be positive");
    if (int rc = make_grid(s->grid, s->dirichlet_kind, S.g)) return rc;
    const int NZ = S.g.NZ, nxy = S.g.NX * S.g.NY;
    if (s->k0 < 0 || s->k1 > NZ || s->k0 >= s->k1) return fail(TL_E_INVALID, "bad slab plane range");
    const int h0 = s->k0 > 0 ? s->k0 - 1 : 0;
    const int h1 = s->k1 < NZ ? s->k1 + 1 : NZ;
    S.own_lo = s->k0 * nxy; S.own_hi = s->k1 * nxy;
    S.st_lo = h0 * nxy; S.st_hi = h1 * nxy;
    const ptrdiff_t base = (ptrdiff_t)S.st_lo;
    S.x = s->x - base; S.b = s->b - base; S.r = s->r - base; S.p0 = s->p0 - base; S.p1 = s->p1 - base;
    S.load = s->load ? s->load - base : nullptr;
    const double V = S.g.h[0] * S.g.h[1] * S.g.h[2];
    for (int a = 0; a < 3; ++a) S.cbase[a] = s->kappa * V / (S.g.h[a] * S.g.h[a]) / 6.0;
    S.mbase = (s->rho_c / s->dt) * V / 24.0;
    S.g_const = s->g_const;
    S.part = s->work;
    S.count = reinterpret_cast<unsigned*>(s->work + 4 * tl::kSlabMaxBlocks);
    S.sums = s->sums;
    int dev = 0;
    TL_CUDA(cudaGetDevice(&dev));
    static int sms_cache[64] = {0};
    if (dev < 0 || dev >= 64) return fail(TL_E_INVALID, "device index");
    if (!sms_cache[dev])
        if (int rc = device_sms(dev, sms_cache[dev])) return rc;
    blocks = 3 * sms_cache[dev];          // flat slab kernels: 3 CTAs per SM
    if (blocks > tl::kSlabMaxBlocks) blocks = tl::kSlabMaxBlocks;
    st = (cudaStream_t)s->stream;
    return TL_OK;
}

// work layout (doubles): [4 kSlabMaxBlocks partials][counter][deposit count][deposit nodes
// kDepMax ints] [control block][item partials 3 kTMaxItems][boundary partials
// 2 kSlabMaxBlocks][tiled arrival counter, item counter]
constexpr int64_t kSlabDepOff = 4 * (int64_t)tl::kSlabMaxBlocks + 1;
constexpr int64_t kSlabCtlOff = (kSlabDepOff + 1 + tl::kDepMax / 2 + 7) / 8 * 8;
constexpr int64_t kSlabIPartOff = kSlabCtlOff + 16;
constexpr int64_t kSlabBPartOff = kSlabIPartOff + 3 * (int64_t)tl::kTMaxItems;
constexpr int64_t kSlabCntOff = kSlabBPartOff + 2 * (int64_t)tl::kSlabMaxBlocks;
static_assert(sizeof(tl::SlabCtl) <= 16 * sizeof(double), "control block");
int64_t tl_slab_work_len(void) { return kSlabCntOff + 2; }

static int slab_dev(const tl_slab* s, tl::SlabDev& D, int& blocks, cudaStream_t& st) {
    if (int rc = slab_params(s, D.S, blocks, st)) return rc;
    if (s->world < 1 || (!s->gath && s->world > 1)) return fail(TL_E_INVALID, "bad slab world / gather buffer");
    // the bulk copies read 16-byte-aligned ranges addressed by global node id
    if ((reinterpret_cast<uintptr_t>(D.S.x) | reinterpret_cast<uintptr_t>(D.S.r) |
         reinterpret_cast<uintptr_t>(D.S.p0) | reinterpret_cast<uintptr_t>(D.S.p1)) & 15)
        return fail(TL_E_INVALID, "slab arrays: the address of global node 0 (x - first stored id) must be "
                                  "16-byte aligned");
    D.k0 = s->k0;
    D.k1 = s->k1;
    D.world = s->world;
    D.gath = s->gath ? s->gath : s->sums;
    D.ctl = reinterpret_cast<tl::SlabCtl*>(s->work + kSlabCtlOff);
    D.ipart = s->work + kSlabIPartOff;
    D.bpart = s->work + kSlabBPartOff;
    D.icount = reinterpret_cast<unsigned*>(s->work + kSlabCntOff);
    D.ictr = reinterpret_cast<unsigned*>(s->work + kSlabCntOff + 1);
    D.nbnd = 0;
    return TL_OK;
}

// planes a neighbour reads (sent after the update): k0 if there is a rank below, k1 - 1 if
// there is one above
static void slab_boundary(const tl_slab* s, int& lo0, int& hi0, int& lo1, int& hi1) {
    const int NZ = s->grid.ncells[2] + 1;
    lo0 = hi0 = lo1 = hi1 = s->k0;
    if (s->k0 > 0) { lo0 = s->k0; hi0 = s->k0 + 1; }
    if (s->k1 < NZ && s->k1 - 1 >= hi0) { lo1 = s->k1 - 1; hi1 = s->k1; }
}

int32_t tl_slab_deposit(const tl_slab* s, const double* points, const double* power, int32_t count) {
    tl::SlabParams S{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_params(s, S, blocks, st)) return rc;
    if (!s->load) return fail(TL_E_INVALID, "slab has no load array");
    if (count < 0 || count * 4 > tl::kDepMax) return fail(TL_E_INVALID, "too many deposit samples");
    if (count > 0 && (!points || !power)) return fail(TL_E_INVALID, "null deposit samples");
    int* prev_n = reinterpret_cast<int*>(s->work + kSlabDepOff);
    int* prev = reinterpret_cast<int*>(s->work + kSlabDepOff + 1);
    tl::k_deposit<<<1, 1024, 0, st>>>(S.g, points, power, count, const_cast<double*>(S.load), prev, prev_n,
                                      S.own_lo, S.own_hi);
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

int32_t tl_slab_begin(const tl_slab* s, const tl_gaussian* src) {
    tl::SlabDev D{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_dev(s, D, blocks, st)) return rc;
    if (!(s->rtol > 0.0) || s->maxiter < 1) return fail(TL_E_INVALID, "bad solver settings");
    tl::k_sd_begin<<<1, 1, 0, st>>>(D.ctl, s->rtol, s->maxiter);
    tl::SlabParams& S = D.S;
    if (src && src->on) {
        S.src.peak = src->peak; S.src.radius = src->radius; S.src.depth = src->depth;
        for (int a = 0; a < 3; ++a) S.src.center[a] = src->center[a];
        S.src.on = 1;
        const size_t smem = gauss_smem(S.g);
        if (smem > 200 * 1024) return fail(TL_E_INVALID, "grid too long for Gaussian tables");
        TL_CUDA(ensure_smem_attr((const void*)tl::k_slab_rhs<true>, smem));
        tl::k_slab_rhs<true><<<blocks, tl::kSlabTPB, smem, st>>>(S);
    } else {
        tl::k_slab_rhs<false><<<blocks, tl::kSlabTPB, 0, st>>>(S);
    }
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

}  // extern "C"
template <class K>
static cudaError_t launch_sd_tiled(K kern, const tl::SlabDev& D, const tl::TPlan& tp, size_t smem, int sms,
                                   cudaStream_t st) {
    cudaError_t e = ensure_smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<sms, (tp.ncw + 1) * 32, smem, st>>>(D, tp);
    return cudaGetLastError();
}
extern "C" {

int32_t tl_slab_direction(const tl_slab* s) {
    tl::SlabDev D{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_dev(s, D, blocks, st)) return rc;
    int dev = 0, sms = 0;
    TL_CUDA(cudaGetDevice(&dev));
    if (int rc = device_sms(dev, sms)) return rc;
    tl::TPlan tp{};
    size_t smem = 0;
    if (!tiled_plan_range(D.S.g, sms, s->k0, s->k1, tp, smem)) return fail(TL_E_INVALID, "no item plan for the slab");
    const bool two = tp.H * D.S.g.NX <= 2 * tp.ncw * 32;
    cudaError_t e = tp.ncw == 16 ? (two ? launch_sd_tiled(tl::k_sd_dir<16, 2>, D, tp, smem, sms, st)
                                        : launch_sd_tiled(tl::k_sd_dir<16, 4>, D, tp, smem, sms, st))
                                 : (two ? launch_sd_tiled(tl::k_sd_dir<19, 2>, D, tp, smem, sms, st)
                                        : launch_sd_tiled(tl::k_sd_dir<19, 4>, D, tp, smem, sms, st));
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("slab direction: ") + cudaGetErrorString(e));
    return TL_OK;
}

int32_t tl_slab_update(const tl_slab* s, int32_t part) {
    tl::SlabDev D{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_dev(s, D, blocks, st)) return rc;
    int lo0, hi0, lo1, hi1;
    slab_boundary(s, lo0, hi0, lo1, hi1);
    if (part == 0) {                       // the planes the neighbours read
        if (hi0 > lo0 || hi1 > lo1) {
            tl::k_sd_upd_flat<<<blocks, tl::kSlabTPB, 0, st>>>(D, lo0, hi0, lo1, hi1);
            TL_CUDA(cudaGetLastError());
        }
        return TL_OK;
    }
    if (part != 1) return fail(TL_E_INVALID, "update part must be 0 (boundary) or 1 (rest)");
    D.nbnd = (hi0 > lo0 || hi1 > lo1) ? blocks : 0;
    const int zlo = hi0 > lo0 ? hi0 : s->k0;
    const int zhi = hi1 > lo1 ? lo1 : s->k1;
    int dev = 0, sms = 0;
    TL_CUDA(cudaGetDevice(&dev));
    if (int rc = device_sms(dev, sms)) return rc;
    tl::TPlan tp{};
    size_t smem = 16;
    if (zhi > zlo) {
        if (!tiled_plan_range(D.S.g, sms, zlo, zhi, tp, smem)) return fail(TL_E_INVALID, "no item plan for the slab");
    } else {
        tp.I = 0;                          // nothing beyond the boundary planes: sum their partials
    }
    if (tp.I == 0) tp.ncw = 16;
    const bool two = tp.I == 0 || tp.H * D.S.g.NX <= 2 * tp.ncw * 32;
    cudaError_t e = tp.ncw == 16 ? (two ? launch_sd_tiled(tl::k_sd_upd<16, 2>, D, tp, smem, sms, st)
                                        : launch_sd_tiled(tl::k_sd_upd<16, 4>, D, tp, smem, sms, st))
                                 : (two ? launch_sd_tiled(tl::k_sd_upd<19, 2>, D, tp, smem, sms, st)
                                        : launch_sd_tiled(tl::k_sd_upd<19, 4>, D, tp, smem, sms, st));
    if (e != cudaSuccess) return fail(TL_E_CUDA, std::string("slab update: ") + cudaGetErrorString(e));
    return TL_OK;
}

int32_t tl_slab_residual(const tl_slab* s) {
    tl::SlabDev D{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_dev(s, D, blocks, st)) return rc;
    tl::k_sd_resid<<<blocks, tl::kSlabTPB, 0, st>>>(D);
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

int32_t tl_slab_finish(const tl_slab* s) {
    tl::SlabDev D{};
    int blocks = 0;
    cudaStream_t st;
    if (int rc = slab_dev(s, D, blocks, st)) return rc;
    tl::k_sd_finish<<<1, 32, 0, st>>>(D);
    TL_CUDA(cudaGetLastError());
    return TL_OK;
}

int32_t tl_slab_poll(const tl_slab* s, int32_t* state, tl_solve_info* info) {
    if (!s || !s->work || !state) return fail(TL_E_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)s->stream;
    tl::SlabCtl c{};
    TL_CUDA(cudaMemcpyAsync(&c, s->work + kSlabCtlOff, sizeof(c), cudaMemcpyDeviceToHost, st));
    TL_CUDA(cudaStreamSynchronize(st));
    *state = c.done;
    if (info) {
        info->iterations = c.status == 1 ? c.maxiter : c.it;
        info->status = c.status;
        info->bnorm = c.bnorm;
        info->rnorm = c.rnorm;
        info->true_resid = c.true_resid;
    }
    return TL_OK;
}

}  // extern "C"
