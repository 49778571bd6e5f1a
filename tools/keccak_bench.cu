// Keccak-f[1600] pipe-balance microbenchmark: Keccak-256 over 4 KB chunks of a
// 512 MB buffer (one thread per chunk, as k_chunk_leaves) for several
// FMA/ALU rotation splits (hash.cuh keccak_f1600_m<MASK>).  Prints GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/keccak_bench tools/keccak_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2510_16028_b200/csrc/common.cuh"
#include "../paper_2510_16028_b200/csrc/hash.cuh"

using namespace nao;

template <uint32_t MASK>
__global__ void __launch_bounds__(128) k_bench(const uint2* __restrict__ data, int64_t nchunks,
                                               int words_per_chunk, uint64_t* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nchunks) return;
    const uint2* p = data + t * (words_per_chunk / 2);
    uint64_t A[25];
#pragma unroll
    for (int i = 0; i < 25; i++) A[i] = 0;
    const int nblk = words_per_chunk / 34;
#pragma unroll 1
    for (int b = 0; b < nblk; b++) {
#pragma unroll
        for (int i = 0; i < 17; i++) {
            const uint2 v = __ldg(p + 17 * b + i);
            A[i] ^= ((uint64_t)v.y << 32) | v.x;
        }
        keccak_f1600_m<MASK>(A);
    }
    out[t] = A[0] ^ A[1] ^ A[2] ^ A[3];
}

template <uint32_t MASK>
void run(const char* name, const uint2* d, int64_t nchunks, int wpc, uint64_t* out, uint64_t* ref) {
    const int blocks = (int)((nchunks + 127) / 128);
    k_bench<MASK><<<blocks, 128>>>(d, nchunks, wpc, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; r++) k_bench<MASK><<<blocks, 128>>>(d, nchunks, wpc, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    uint64_t h[4];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    bool same = true;
    if (ref[0] == 0 && ref[1] == 0) { for (int i = 0; i < 4; i++) ref[i] = h[i]; }
    else for (int i = 0; i < 4; i++) same &= (ref[i] == h[i]);
    const double bytes = (double)nchunks * (wpc / 34) * 136;
    printf("{\"variant\": \"%s\", \"mask\": \"0x%08x\", \"ms\": %.4f, \"GB/s\": %.1f, \"same\": %s}\n",
           name, MASK, ms, bytes / (ms * 1e-3) / 1e9, same ? "true" : "false");
}

int main() {
    const int wpc = 1020;  // 30 Keccak blocks (4080 B) per chunk
    const int64_t nchunks = (512ll << 20) / (wpc * 4);
    uint2* d;
    uint64_t* out;
    cudaMalloc(&d, nchunks * wpc * 4);
    cudaMalloc(&out, nchunks * 8);
    cudaMemset(d, 0x5a, nchunks * wpc * 4);
    uint64_t ref[4] = {0, 0, 0, 0};
    run<0x00000000u>("alu-only", d, nchunks, wpc, out, ref);
    run<0x1F000000u>("theta-fma", d, nchunks, wpc, out, ref);
    run<0x00000FFFu>("rho12-fma", d, nchunks, wpc, out, ref);
    run<0x00555555u>("rho-alt12", d, nchunks, wpc, out, ref);
    run<0x1F000FFFu>("theta+rho12", d, nchunks, wpc, out, ref);
    run<0x00FFFFFFu>("rho-all", d, nchunks, wpc, out, ref);
    run<0x1FFFFFFFu>("all-fma", d, nchunks, wpc, out, ref);
    run<0x000000FFu>("rho8", d, nchunks, wpc, out, ref);
    run<0x0000FFFFu>("rho16", d, nchunks, wpc, out, ref);
    run<0x9F000000u>("w32-theta", d, nchunks, wpc, out, ref);
    run<0x80000FFFu>("w32-rho12", d, nchunks, wpc, out, ref);
    run<0x9F000FFFu>("w32-theta+rho12", d, nchunks, wpc, out, ref);
    run<0x80FFFFFFu>("w32-rho-all", d, nchunks, wpc, out, ref);
    run<0x9FFFFFFFu>("w32-all", d, nchunks, wpc, out, ref);
    run<0x8000FFFFu>("w32-rho16", d, nchunks, wpc, out, ref);
    run<0x80555555u>("w32-rho-alt12", d, nchunks, wpc, out, ref);
    run<0x00000000u>("alu-only-again", d, nchunks, wpc, out, ref);
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
