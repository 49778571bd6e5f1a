// Throughput of the FP64 / conversion pipes on this part (ops per clock per SM):
// DADD, DMUL, DFMA, F2F.F64.F32, F2F.F32.F64, FADD (reference), 8 independent chains
// per thread, 148 x 1024 threads.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
    double d[8]; float f[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { d[i] = threadIdx.x * 1e-3 + i; f[i] = threadIdx.x * 1e-3f + i; }
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) d[i] = __dadd_rn(d[i], 1.0000001);
            if (OP == 1) d[i] = __dmul_rn(d[i], 1.0000001);
            if (OP == 2) d[i] = __fma_rn(d[i], 1.0000001, 1e-9);
            if (OP == 3) { d[i] = (double)f[i]; f[i] = __fadd_rn(f[i], (float)d[(i + 1) & 7]); }
            if (OP == 4) { f[i] = __double2float_rn(d[i]); d[i] = __dadd_rn(d[i], (double)1); }
            if (OP == 5) f[i] = __fadd_rn(f[i], 1.0000001f);
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += (float)d[i] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
template <int OP> void run(const char* name) {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
    const int iters = 4096;
    k<OP><<<148, 1024>>>(o, 16, c);
    cudaDeviceSynchronize();
    k<OP><<<148, 1024>>>(o, iters, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double ops = 1024.0 * iters * 8;  // per SM (one block per SM)
    printf("{\"op\": \"%s\", \"ops_per_clk_per_sm\": %.1f}\n", name, ops / h);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<0>("DADD"); run<1>("DMUL"); run<2>("DFMA"); run<3>("F2F.F64.F32 (+FADD)");
    run<4>("F2F.F32.F64 (+DADD)"); run<5>("FADD");
    return 0;
}
