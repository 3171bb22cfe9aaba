// bulkbench.cu — HBM read throughput of a cp.async.bulk ring (one producer lane per CTA,
// consumer warps reading each stage from shared memory), the data path of k_t_cg.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulkbench tools/bulkbench.cu
// Sweeps chunk size, 16-byte misalignment, ring depth and CTAs per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
    unsigned d;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(d) : "r"(sa(b)), "r"(par) : "memory");
    } while (!d);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(n), "r"(sa(b)) : "memory");
}

extern __shared__ __align__(128) double sm[];

// Chunk c of the array (chunk doubles each, offset by mis doubles) goes to CTA c % G.
__global__ void k_bulk(const double* a, long long nchunks, int chunk, int mis, int NS, int ncopy, double* out) {
    __shared__ uint64_t full[32], empty[32];
    const int ncw = blockDim.x / 32 - 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], ncw); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int w = threadIdx.x / 32;
    const int stage = chunk + 16;
    double acc = 0.0;
    if (w == ncw) {
        if ((threadIdx.x & 31) == 0) {
            unsigned t = 0;
            for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++t) {
                const int s = t % NS;
                mb_wait(&empty[s], ((t / NS) & 1) ^ 1);
                const unsigned bytes = chunk * 8;
                mb_arrive_tx(&full[s], bytes);
                const int per = chunk / ncopy;
                for (int q = 0; q < ncopy; ++q)
                    bulk(sm + (size_t)s * stage + q * per, a + c * chunk + mis + q * per, per * 8, &full[s]);
            }
        }
    } else {
        unsigned t = 0;
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++t) {
            const int s = t % NS;
            mb_wait(&full[s], (t / NS) & 1);
            for (int e = threadIdx.x; e < chunk; e += ncw * 32) acc += sm[(size_t)s * stage + e];
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mb_arrive(&empty[s]);
        }
    }
    if (acc == 12345.0) *out = acc;
}

__global__ void k_copy(const double* a, double* b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1LL << 29;                 // 4 GiB of doubles
    double *a, *b, *out;
    cudaMalloc(&a, (n + 64) * 8);
    cudaMalloc(&b, n * 8);
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, (n + 64) * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    k_copy<<<sms * 4, 512>>>(a, b, n);
    cudaEventRecord(e0);
    k_copy<<<sms * 4, 512>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy kernel: %.0f GB/s (read+write)\n", 2.0 * n * 8 / ms / 1e6);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const int chunks[] = {1024, 2048, 4096, 8192};
    for (int cpb : {1, 2}) {
        for (int chunk : chunks) {
            for (int mis : {0, 2}) {
                for (int ncw : {4, 16}) {
                    for (int ncopy : {1, 4}) {
                        const size_t stage_b = (size_t)(chunk + 16) * 8;
                        int NS = (int)((220 * 1024 / cpb) / stage_b);
                        if (NS > 16) NS = 16;
                        if (NS < 2) continue;
                        const long long nch = (n - 64) / chunk;
                        const size_t smem = NS * stage_b;
                        k_bulk<<<sms * cpb, (ncw + 1) * 32, smem>>>(a, nch, chunk, mis, NS, ncopy, out);
                        cudaEventRecord(e0);
                        k_bulk<<<sms * cpb, (ncw + 1) * 32, smem>>>(a, nch, chunk, mis, NS, ncopy, out);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        cudaError_t err = cudaGetLastError();
                        cudaEventElapsedTime(&ms, e0, e1);
                        printf("ctas/SM %d chunk %5d B mis %2d B consumers %2d warps copies %d NS %2d: %6.0f GB/s %s\n",
                               cpb, chunk * 8, mis * 8, ncw, ncopy, NS, nch * chunk * 8.0 / ms / 1e6,
                               err == cudaSuccess ? "" : cudaGetErrorString(err));
                    }
                }
            }
        }
    }
    return 0;
}
