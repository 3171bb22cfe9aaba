// syncbench.cu — microbenchmark of grid-wide barriers on B200 (design input for k_pcg).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o syncbench tools/syncbench.cu
// Measures per-barrier latency of cooperative_groups grid.sync() and of a
// hand-written sense-reversal barrier (one red.release + ld.acquire spin per block)
// for 1..4 blocks per SM, plus the cost of a 148-partial fixed-order reduction.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* part, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) part[blockIdx.x] = it + blockIdx.x;
        g.sync();
        if (threadIdx.x < 32) {
            double s = 0.0;
            for (int b = threadIdx.x; b < gridDim.x; b += 32) s += __ldcg(part + b);
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            acc += s;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

__device__ __forceinline__ void bar_arrive_wait(unsigned* count, volatile unsigned* gen, unsigned nblocks,
                                                unsigned& my_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g0 = my_gen;
        __threadfence();
        unsigned prev = atomicAdd(count, 1u);
        if (prev == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicExch((unsigned*)gen, g0 + 1);
        } else {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
            } while (v == g0);
        }
        my_gen = g0 + 1;
    }
    __syncthreads();
}

__global__ void k_custom(int iters, double* part, double* out, unsigned* count, unsigned* gen) {
    __shared__ unsigned my_gen;
    if (threadIdx.x == 0) my_gen = *((volatile unsigned*)gen);
    __syncthreads();
    unsigned mg = my_gen;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) part[blockIdx.x] = it + blockIdx.x;
        bar_arrive_wait(count, gen, gridDim.x, mg);
        if (threadIdx.x < 32) {
            double s = 0.0;
            for (int b = threadIdx.x; b < gridDim.x; b += 32) s += __ldcg(part + b);
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            acc += s;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

__global__ void k_empty() {}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *part, *out;
    unsigned *count, *gen;
    cudaMalloc(&part, 8 * 4096);
    cudaMalloc(&out, 8);
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(count, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int tpb : {256, 512, 1024}) {
        for (int per = 1; per <= 4; ++per) {
            if (tpb * per > 2048) continue;
            int nb = per * sms;
            void* args[] = {(void*)&iters, &part, &out};
            cudaLaunchCooperativeKernel((void*)k_cg, nb, tpb, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, nb, tpb, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms_cg = 0;
            cudaEventElapsedTime(&ms_cg, a, b);
            void* args2[] = {(void*)&iters, &part, &out, &count, &gen};
            cudaLaunchCooperativeKernel((void*)k_custom, nb, tpb, args2, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_custom, nb, tpb, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms_c = 0;
            cudaEventElapsedTime(&ms_c, a, b);
            cudaError_t e = cudaGetLastError();
            printf("tpb=%4d blocks=%4d  cg.sync+reduce %.3f us   custom barrier+reduce %.3f us  %s\n", tpb, nb,
                   1e3 * ms_cg / iters, 1e3 * ms_c / iters, cudaGetErrorString(e));
        }
    }
    // back-to-back dependent launches (stream) for comparison
    cudaEventRecord(a);
    for (int i = 0; i < 2000; ++i) k_empty<<<sms, 256>>>();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel launch (stream, back to back): %.3f us\n", 1e3 * ms / 2000);
    return 0;
}
