// Measured integer-ALU peaks for the commit roofline (bench.py reads
// profiles/r2_alu_peak.json):
//   * LOP3 and SHF.L.W (funnel shift) throughput, ops / clk / SM, from
//     independent register chains (no memory);
//   * the compute-only Keccak-f[1600] rate of this library's own permutation
//     (csrc/hash.cuh keccak_f1600, state in registers, no loads) on every SM,
//     timed with CUDA events at the clocks the GPU runs -> bytes/s of rate
//     (136 B per permutation): the ceiling of the fused commit's sponge.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include tools/alu_peak.cu -o tools/alu_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2510_16028_b200/csrc/common.cuh"
#include "../paper_2510_16028_b200/csrc/hash.cuh"

template <int OP>
__global__ void k_pipe(uint32_t* out, int iters, long long* clk) {
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 8; i++) r[i] = threadIdx.x * 2654435761u + i;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) {  // LOP3: a ^ (~b & c)
                uint32_t d;
                asm volatile("lop3.b32 %0, %1, %2, %3, 0xD2;" : "=r"(d) : "r"(r[i]), "r"(r[(i + 1) & 7]), "r"(r[(i + 2) & 7]));
                r[i] = d;
            } else {  // SHF.L.W funnel rotate
                r[i] = __funnelshift_l(r[i], r[(i + 3) & 7], 7);
            }
        }
    }
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

__global__ void __launch_bounds__(128, 4) k_keccak(uint64_t* out, int perms) {
    uint64_t A[25];
#pragma unroll
    for (int i = 0; i < 25; i++) A[i] = (uint64_t)(threadIdx.x + blockIdx.x * 977u) * (i + 1);
    for (int p = 0; p < perms; p++) nao::keccak_f1600(A);
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 25; i++) s ^= A[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
double pipe_rate(int iters) {
    uint32_t* o; long long* c;
    cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
    k_pipe<OP><<<148, 1024>>>(o, 16, c);
    cudaDeviceSynchronize();
    k_pipe<OP><<<148, 1024>>>(o, iters, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    cudaFree(o); cudaFree(c);
    return 1024.0 * iters * 8 / (double)h;  // one block per SM
}

int main() {
    const double lop3 = pipe_rate<0>(4096), shf = pipe_rate<1>(4096);
    uint64_t* o;
    const int ctas = 148 * 4, threads = 128, perms = 2048;
    cudaMalloc(&o, (size_t)ctas * threads * 8);
    k_keccak<<<ctas, threads>>>(o, 8);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        k_keccak<<<ctas, threads>>>(o, perms);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double nperm = (double)ctas * threads * perms;
    const double gbs = nperm * 136.0 / (best * 1e-3) / 1e9;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"lop3_ops_per_clk_per_sm\": %.1f, \"shf_ops_per_clk_per_sm\": %.1f, "
           "\"keccak_f1600_perms_per_s\": %.4g, \"keccak_rate_gbs\": %.1f, "
           "\"keccak_ms\": %.3f, \"ctas\": %d, \"threads\": %d, \"perms_per_thread\": %d, "
           "\"attr_clock_mhz\": %.0f}\n",
           lop3, shf, nperm / (best * 1e-3), gbs, best, ctas, threads, perms, clk_khz / 1e3);
    return 0;
}
