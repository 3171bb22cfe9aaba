// streambench.cu — HBM microbenchmark of the streaming CG sweep shapes (sm_100a, fp64).
// Not part of the product: isolates the memory behaviour of the two CG sweeps from the
// CG control logic.  All nodes are treated as interior (constant 7-point weights).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/streambench tools/streambench.cu
//   tools/streambench NX NY NZ
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ double g_sink[1];

// copy: read 1 write 1 (the MEASURED_PEAKS reference shape)
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, long n) {
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) b[p] = a[p];
}
// stream B shape without stencil: read 3 write 2
__global__ void k_r3w2(const double* __restrict__ p_, double* __restrict__ x, double* __restrict__ r, long n, double al) {
    double acc = 0;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        double pv = p_[p];
        double xv = x[p] + al * pv, rv = r[p] - al * pv;
        x[p] = xv; r[p] = rv; acc += rv * rv;
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

// B1: grid-stride, thread per node, 7-point stencil of p from global, x, r updated
__global__ void k_b1(const double* __restrict__ pp, double* __restrict__ x, double* __restrict__ r, int NX, int NY,
                     int NZ, double al) {
    const long sz = (long)NX * NY, n = sz * NZ;
    double acc = 0;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        if (p < sz || p >= n - sz) continue;
        const double c = pp[p];
        const double q = 6.1 * c - ((0.9 * (pp[p - 1] + pp[p + 1]) + 0.8 * (pp[p - NX] + pp[p + NX])) + 0.7 * (pp[p - sz] + pp[p + sz]));
        const double xv = x[p] + al * c, rv = r[p] - al * q;
        x[p] = xv; r[p] = rv; acc += rv * rv;
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

// A1: grid-stride, p = z + beta pold recomputed at 7 points (14 loads), p written, p.q
__global__ void k_a1(const double* __restrict__ r, const double* __restrict__ po, double* __restrict__ pn, int NX,
                     int NY, int NZ, double be) {
    const long sz = (long)NX * NY, n = sz * NZ;
    double acc = 0;
    auto P = [&](long q) { return 0.25 * r[q] + be * po[q]; };
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        if (p < sz || p >= n - sz) continue;
        const double c = P(p);
        const double q = 6.1 * c - ((0.9 * (P(p - 1) + P(p + 1)) + 0.8 * (P(p - NX) + P(p + NX))) + 0.7 * (P(p - sz) + P(p + sz)));
        pn[p] = c; acc += c * q;
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

// A2: forward edges only: p.Ap = sum diag p^2 - 2 sum c p_i p_j over +x, +y, +z (8 loads)
__global__ void k_a2(const double* __restrict__ r, const double* __restrict__ po, double* __restrict__ pn, int NX,
                     int NY, int NZ, double be) {
    const long sz = (long)NX * NY, n = sz * NZ;
    double acc = 0;
    auto P = [&](long q) { return 0.25 * r[q] + be * po[q]; };
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        if (p >= n - sz) continue;
        const double c = P(p);
        acc += c * (6.1 * c - 2.0 * (0.9 * P(p + 1) + 0.8 * P(p + NX) + 0.7 * P(p + sz)));
        pn[p] = c;
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

// Row march: a CTA owns a full row j (threads cover x) and a z chunk; z neighbours in
// registers, x neighbours from the thread's own row loads (L1), y rows j±1 loaded.
__global__ void k_brow(const double* __restrict__ pp, double* __restrict__ x, double* __restrict__ r, int NX, int NY,
                       int NZ, int zlen, double al) {
    const long sz = (long)NX * NY;
    double acc = 0;
    const int nzc = (NZ + zlen - 1) / zlen;
    for (int u = blockIdx.x; u < NY * nzc; u += gridDim.x) {
        const int j = u % NY, kc = u / NY;
        if (j == 0 || j == NY - 1) continue;
        const int ka = max(1, kc * zlen), kb = min(NZ - 1, kc * zlen + zlen);
        for (int i = threadIdx.x + 1; i < NX - 1; i += blockDim.x) {
            long p = (long)(ka)*sz + (long)j * NX + i;
            double zm = pp[p - sz], c = pp[p];
            for (int k = ka; k < kb; ++k, p += sz) {
                const double zp = pp[p + sz];
                const double q = 6.1 * c - ((0.9 * (pp[p - 1] + pp[p + 1]) + 0.8 * (pp[p - NX] + pp[p + NX])) + 0.7 * (zm + zp));
                const double xv = x[p] + al * c, rv = r[p] - al * q;
                x[p] = xv; r[p] = rv; acc += rv * rv;
                zm = c; c = zp;
            }
        }
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

// Plane-parallel z march: each thread owns an (i, j) column, the CTAs cover a plane's
// rows contiguously (thread index = i + NX j over the plane), march a z chunk.
__global__ void k_bcol(const double* __restrict__ pp, double* __restrict__ x, double* __restrict__ r, int NX, int NY,
                       int NZ, int zlen, double al) {
    const long sz = (long)NX * NY;
    double acc = 0;
    const int nzc = (NZ + zlen - 1) / zlen;
    const long ncol = sz;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < ncol * nzc; u += (long)gridDim.x * blockDim.x) {
        const long col = u % ncol;
        const int kc = (int)(u / ncol);
        const int i = (int)(col % NX), j = (int)(col / NX);
        if (i == 0 || i == NX - 1 || j == 0 || j == NY - 1) continue;
        const int ka = max(1, kc * zlen), kb = min(NZ - 1, kc * zlen + zlen);
        long p = (long)ka * sz + col;
        double zm = pp[p - sz], c = pp[p];
        for (int k = ka; k < kb; ++k, p += sz) {
            const double zp = pp[p + sz];
            const double q = 6.1 * c - ((0.9 * (pp[p - 1] + pp[p + 1]) + 0.8 * (pp[p - NX] + pp[p + NX])) + 0.7 * (zm + zp));
            const double xv = x[p] + al * c, rv = r[p] - al * q;
            x[p] = xv; r[p] = rv; acc += rv * rv;
            zm = c; c = zp;
        }
    }
    if (acc == 12345.0) g_sink[0] = acc;
}

static float timeit(void (*launch)(void*), void* ctx, int reps, double* flush, long nflush) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f, tot = 0;
    for (int t = 0; t < reps + 1; ++t) {
        cudaMemsetAsync(flush, t, nflush * 8);
        cudaEventRecord(a);
        launch(ctx);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (t > 0) { tot += ms; if (ms < best) best = ms; }
    }
    CK(cudaGetLastError());
    return tot / reps;
}

struct Ctx { double *a, *b, *c, *d; int NX, NY, NZ; long n; int grid, tpb, zlen; };
static Ctx C;

int main(int argc, char** argv) {
    C.NX = argc > 1 ? atoi(argv[1]) : 301;
    C.NY = argc > 2 ? atoi(argv[2]) : 301;
    C.NZ = argc > 3 ? atoi(argv[3]) : 76;
    C.n = (long)C.NX * C.NY * C.NZ;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    CK(cudaMalloc(&C.a, C.n * 8)); CK(cudaMalloc(&C.b, C.n * 8)); CK(cudaMalloc(&C.c, C.n * 8)); CK(cudaMalloc(&C.d, C.n * 8));
    cudaMemset(C.a, 0, C.n * 8); cudaMemset(C.b, 0, C.n * 8); cudaMemset(C.c, 0, C.n * 8); cudaMemset(C.d, 0, C.n * 8);
    long nflush = 40l << 20;   // 320 MB > L2
    double* flush; CK(cudaMalloc(&flush, nflush * 8));
    printf("grid %d x %d x %d = %ld nodes, %d SMs\n", C.NX, C.NY, C.NZ, C.n, sms);
    const double GB = 1e9;
    for (int tpb : {256, 512}) {
        for (int per : {2, 4, 8}) {
            C.grid = sms * per; C.tpb = tpb;
            if (tpb * per > 2048) continue;
            float t;
            t = timeit([](void*) { k_copy<<<C.grid, C.tpb>>>(C.a, C.b, C.n); }, nullptr, 5, flush, nflush);
            printf("tpb %3d x%d  copy   %7.1f us %6.0f GB/s\n", tpb, per, t * 1e3, 16.0 * C.n / (t * 1e-3) / GB);
            t = timeit([](void*) { k_r3w2<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.n, 0.5); }, nullptr, 5, flush, nflush);
            printf("tpb %3d x%d  r3w2   %7.1f us %6.0f GB/s\n", tpb, per, t * 1e3, 40.0 * C.n / (t * 1e-3) / GB);
            t = timeit([](void*) { k_b1<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.NX, C.NY, C.NZ, 0.5); }, nullptr, 5, flush, nflush);
            printf("tpb %3d x%d  B1     %7.1f us %6.0f GB/s\n", tpb, per, t * 1e3, 40.0 * C.n / (t * 1e-3) / GB);
            t = timeit([](void*) { k_a1<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.NX, C.NY, C.NZ, 0.5); }, nullptr, 5, flush, nflush);
            printf("tpb %3d x%d  A1     %7.1f us %6.0f GB/s\n", tpb, per, t * 1e3, 24.0 * C.n / (t * 1e-3) / GB);
            t = timeit([](void*) { k_a2<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.NX, C.NY, C.NZ, 0.5); }, nullptr, 5, flush, nflush);
            printf("tpb %3d x%d  A2     %7.1f us %6.0f GB/s\n", tpb, per, t * 1e3, 24.0 * C.n / (t * 1e-3) / GB);
            for (int zl : {8, 16, 32, 1 << 20}) {
                C.zlen = zl;
                t = timeit([](void*) { k_brow<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.NX, C.NY, C.NZ, C.zlen, 0.5); }, nullptr, 5, flush, nflush);
                printf("tpb %3d x%d  Brow z%-7d %7.1f us %6.0f GB/s\n", tpb, per, zl, t * 1e3, 40.0 * C.n / (t * 1e-3) / GB);
                t = timeit([](void*) { k_bcol<<<C.grid, C.tpb>>>(C.a, C.b, C.c, C.NX, C.NY, C.NZ, C.zlen, 0.5); }, nullptr, 5, flush, nflush);
                printf("tpb %3d x%d  Bcol z%-7d %7.1f us %6.0f GB/s\n", tpb, per, zl, t * 1e3, 40.0 * C.n / (t * 1e-3) / GB);
            }
        }
    }
    return 0;
}
