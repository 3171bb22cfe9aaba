// syncbench2.cu — all-reduce-with-barrier variants for the SMEM-resident CG loop (one
// reduction of 3 doubles over 148 CTAs per iteration):
//   A: the round-1/2 grid_allreduce (partials + red.release counter + ld.acquire poll + reload)
//   B: flagged words ("LL": every 8-byte word = 4 data bytes + 4-byte epoch), all CTAs poll
//      all slots; a fence.acq_rel.gpu before the stores orders the CTA's earlier global stores
//   C: B without the fence (lower bound; not usable where surface data must be ordered)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o syncbench2 tools/syncbench2.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NV>
__device__ __forceinline__ void allred_a(double (&v)[NV], double* red, double* part, int G, unsigned* cnt,
                                         unsigned target, double* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
        for (int k = 0; k < NV; ++k) red[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
        double sv[NV];
        for (int k = 0; k < NV; ++k) sv[k] = warp_sum(lane < nw ? red[k * 32 + lane] : 0.0);
        if (lane == 0) {
            for (int k = 0; k < NV; ++k) part[k * G + blockIdx.x] = sv[k];
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        }
        unsigned c;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(cnt) : "memory");
        } while ((int)(c - target) < 0);
        for (int k = 0; k < NV; ++k) {
            double acc = 0.0;
            for (int t = 0; t < 5; ++t) {
                const int bb = lane + 32 * t;
                acc += bb < G ? __ldcg(part + k * G + bb) : 0.0;
            }
            acc = warp_sum(acc);
            if (lane == 0) tot[k] = acc;
        }
    }
    __syncthreads();
}

// slots: [parity][G][2*NV] 8-byte words {lo/hi 32 data bits, epoch}
template <int NV, bool FENCE>
__device__ __forceinline__ void allred_ll(double (&v)[NV], double* red, unsigned long long* slots, int G,
                                          unsigned epoch, double* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
        for (int k = 0; k < NV; ++k) red[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
        unsigned long long* base = slots + (size_t)(epoch & 1u) * G * 2 * NV;
        double sv[NV];
        for (int k = 0; k < NV; ++k) sv[k] = warp_sum(lane < nw ? red[k * 32 + lane] : 0.0);
        if (FENCE) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (lane < 2 * NV) {
            double x = sv[0];
            for (int k = 1; k < NV; ++k) x = (lane >> 1) == k ? sv[k] : x;
            const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
            const unsigned half = (lane & 1) ? (unsigned)(bits >> 32) : (unsigned)bits;
            const unsigned long long word = ((unsigned long long)epoch << 32) | half;
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(base + (size_t)blockIdx.x * 2 * NV + lane), "l"(word) : "memory");
        }
        // poll: the G * NV 16-byte units are contiguous; lane takes units lane, lane + 32, ...
        // (all loads of a round in flight together; unit u = CTA u / NV, value u % NV)
        constexpr int PU = (160 * NV + 31) / 32;
        const int nu = G * NV;
        unsigned long long wa[PU], wb[PU];
        bool all;
        do {
            all = true;
#pragma unroll
            for (int t = 0; t < PU; ++t) {
                const int u = lane + 32 * t;
                if (u < nu)
                    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(wa[t]), "=l"(wb[t]) : "l"(base + 2 * u) : "memory");
            }
#pragma unroll
            for (int t = 0; t < PU; ++t) {
                const int u = lane + 32 * t;
                if (u < nu) all = all && (unsigned)(wa[t] >> 32) == epoch && (unsigned)(wb[t] >> 32) == epoch;
            }
        } while (!__all_sync(0xffffffffu, all));
        // fixed-order sums: value k of CTA c sits in unit c * NV + k; stage through smem
        double acc[NV];
#pragma unroll
        for (int t = 0; t < PU; ++t) {
            const int u = lane + 32 * t;
            if (u < nu) red[256 + u] = __longlong_as_double((long long)((wa[t] & 0xffffffffull) | (wb[t] << 32)));
        }
        __syncwarp();
        for (int k = 0; k < NV; ++k) {
            acc[k] = 0.0;
            for (int t = 0; t < 5; ++t) {
                const int bb = lane + 32 * t;
                if (bb < G) acc[k] += red[256 + bb * NV + k];
            }
        }
        if (FENCE) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int k = 0; k < NV; ++k) {
            const double s = warp_sum(acc[k]);
            if (lane == 0) tot[k] = s;
        }
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_bench(int iters, double* part, unsigned long long* slots, unsigned* cnt,
                                                  double* surf, double* out) {
    __shared__ double red[8 * 32 + 160 * 3];
    __shared__ double tot[8];
    const int G = gridDim.x;
    unsigned target = __ldcg(cnt);
    unsigned epoch = __ldcg(cnt + 1);
    cg::this_grid().sync();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[3] = {1.0 + threadIdx.x + it, 2.0 * blockIdx.x, 0.5 * it};
        // surface exchange stand-in: one store per thread of the first two warps
        if (threadIdx.x < 64) surf[(size_t)(it & 1) * G * 64 + blockIdx.x * 64 + threadIdx.x] = v[0];
        if (MODE == 0) {
            target += (unsigned)G;
            allred_a<3>(v, red, part + (size_t)(it & 1) * 3 * G, G, cnt, target, tot);
        } else {
            ++epoch;
            allred_ll<3, MODE == 1>(v, red, slots, G, epoch, tot);
        }
        acc += tot[0] + tot[1] + tot[2];
        // read a neighbour's surface value (checks the ordering the fence is for)
        const int nbq = (blockIdx.x + 1) % G;
        if (threadIdx.x < 64) {
            const double s = __ldcg(surf + (size_t)(it & 1) * G * 64 + nbq * 64 + threadIdx.x);
            if (s != 1.0 + threadIdx.x + it) acc = -1e300;
        }
    }
    cg::this_grid().sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *out = acc;
        if (MODE != 0) cnt[1] = epoch;
    }
}

// D: every CTA pushes its flagged words to a private region of every CTA (no hot lines: a CTA
// polls only its own G * 2 * NV words), and the surface exchange uses flagged words too, so no
// fence is needed anywhere.  slots: [parity][dest G][src G][2*NV]
template <int NV>
__device__ __forceinline__ void allred_push(double (&v)[NV], double* red, unsigned long long* slots, int G,
                                            unsigned epoch, double* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
        for (int k = 0; k < NV; ++k) red[k * 32 + wid] = v[k];
    __syncthreads();
    unsigned long long* base = slots + (size_t)(epoch & 1u) * G * G * 2 * NV;
    // all warps: block totals (each warp recomputes them), then the G * 2 * NV pushes spread over the CTA
    double sv[NV];
    for (int k = 0; k < NV; ++k) sv[k] = warp_sum(lane < nw ? red[k * 32 + lane] : 0.0);
    for (int q = threadIdx.x; q < G * 2 * NV; q += blockDim.x) {
        const int dest = q / (2 * NV), wq = q % (2 * NV);
        double x = sv[0];
        for (int k = 1; k < NV; ++k) x = (wq >> 1) == k ? sv[k] : x;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
        const unsigned half = (wq & 1) ? (unsigned)(bits >> 32) : (unsigned)bits;
        const unsigned long long word = ((unsigned long long)epoch << 32) | half;
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(base + ((size_t)dest * G + blockIdx.x) * 2 * NV + wq), "l"(word) : "memory");
    }
    if (wid == 0) {
        const unsigned long long* mine = base + (size_t)blockIdx.x * G * 2 * NV;
        constexpr int PU = (160 * NV + 31) / 32;
        const int nu = G * NV;
        unsigned long long wa[PU], wb[PU];
        bool all;
        do {
            all = true;
#pragma unroll
            for (int t = 0; t < PU; ++t) {
                const int u = lane + 32 * t;
                if (u < nu)
                    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(wa[t]), "=l"(wb[t]) : "l"(mine + 2 * u) : "memory");
            }
#pragma unroll
            for (int t = 0; t < PU; ++t) {
                const int u = lane + 32 * t;
                if (u < nu) all = all && (unsigned)(wa[t] >> 32) == epoch && (unsigned)(wb[t] >> 32) == epoch;
            }
        } while (!__all_sync(0xffffffffu, all));
#pragma unroll
        for (int t = 0; t < PU; ++t) {
            const int u = lane + 32 * t;
            if (u < nu) red[256 + u] = __longlong_as_double((long long)((wa[t] & 0xffffffffull) | (wb[t] << 32)));
        }
        __syncwarp();
        for (int k = 0; k < NV; ++k) {
            double acc = 0.0;
            for (int t = 0; t < 5; ++t) {
                const int bb = lane + 32 * t;
                if (bb < G) acc += red[256 + bb * NV + k];
            }
            acc = warp_sum(acc);
            if (lane == 0) tot[k] = acc;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(512, 1) k_bench_push(int iters, unsigned long long* slots, unsigned* cnt,
                                                       unsigned long long* surf, double* out) {
    __shared__ double red[8 * 32 + 160 * 3];
    __shared__ double tot[8];
    const int G = gridDim.x;
    unsigned epoch = __ldcg(cnt + 1);
    cg::this_grid().sync();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[3] = {1.0 + threadIdx.x + it, 2.0 * blockIdx.x, 0.5 * it};
        ++epoch;
        // surface exchange stand-in with flagged words: 4 doubles per thread (2048 per CTA)
        for (int q = 0; q < 4; ++q) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(v[0] + q);
            unsigned long long* d = surf + ((size_t)(epoch & 1u) * G * 2048 + blockIdx.x * 2048 + q * 512 + threadIdx.x) * 2;
            asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(((unsigned long long)epoch << 32) | (unsigned)bits),
                         "l"(((unsigned long long)epoch << 32) | (unsigned)(bits >> 32)) : "memory");
        }
        allred_push<3>(v, red, slots, G, epoch, tot);
        acc += tot[0] + tot[1] + tot[2];
        const int nbq = (blockIdx.x + 1) % G;
        unsigned long long a[4], b[4];
        bool all;
        do {
            all = true;
            for (int q = 0; q < 4; ++q) {
                const unsigned long long* d = surf + ((size_t)(epoch & 1u) * G * 2048 + nbq * 2048 + q * 512 + threadIdx.x) * 2;
                asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a[q]), "=l"(b[q]) : "l"(d) : "memory");
            }
            for (int q = 0; q < 4; ++q) all = all && (unsigned)(a[q] >> 32) == epoch && (unsigned)(b[q] >> 32) == epoch;
        } while (!all);
        for (int q = 0; q < 4; ++q) {
            const double sval = __longlong_as_double((long long)((a[q] & 0xffffffffull) | (b[q] << 32)));
            if (sval != 1.0 + threadIdx.x + it + q) acc = -1e300;
        }
    }
    cg::this_grid().sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *out = acc;
        cnt[1] = epoch;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *part, *out, *surf;
    unsigned long long* slots;
    unsigned* cnt;
    cudaMalloc(&part, 8 * 4096);
    cudaMalloc(&slots, 8 * 2 * 160 * 8);
    cudaMalloc(&surf, 8 * 2 * 160 * 64);
    cudaMalloc(&out, 8);
    cudaMalloc(&cnt, 8);
    cudaMemset(cnt, 0, 8);
    cudaMemset(slots, 0, 8 * 2 * 160 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4000;
    const char* names[3] = {"A counter+partials (current)", "B flagged words + fences", "C flagged words, no fence"};
    void* fns[3] = {(void*)k_bench<0>, (void*)k_bench<1>, (void*)k_bench<2>};
    for (int rep = 0; rep < 2; ++rep)
        for (int m = 0; m < 3; ++m) {
            void* args[] = {&iters, &part, &slots, &cnt, &surf, &out};
            cudaLaunchCooperativeKernel(fns[m], sms, 512, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fns[m], sms, 512, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            double h = 0;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("%-32s %.3f us per all-reduce (%d CTAs x 512)  check %s  %s\n", names[m], 1e3 * ms / iters, sms,
                   h > 0 ? "ok" : "ORDER VIOLATION", cudaGetErrorString(cudaGetLastError()));
        }
    {
        unsigned long long *pslots, *psurf;
        cudaMalloc(&pslots, (size_t)8 * 2 * 160 * 160 * 6);
        cudaMalloc(&psurf, (size_t)16 * 2 * 160 * 2048);
        cudaMemset(pslots, 0, (size_t)8 * 2 * 160 * 160 * 6);
        cudaMemset(psurf, 0, (size_t)16 * 2 * 160 * 2048);
        for (int rep = 0; rep < 3; ++rep) {
            void* args[] = {&iters, &pslots, &cnt, &psurf, &out};
            cudaLaunchCooperativeKernel((void*)k_bench_push, sms, 512, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_bench_push, sms, 512, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            double h = 0;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("%-32s %.3f us per all-reduce + 2048-double flagged surface exchange  check %s  %s\n",
                   "D push-to-all flagged words", 1e3 * ms / iters, h > 0 ? "ok" : "ORDER VIOLATION",
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
