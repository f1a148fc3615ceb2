// Microbenchmark: tcgen05.mma throughput for the conditioning kernel's shapes
// (M=128, N=64/128/256, K=16, bf16 -> f32), A from TMEM (ts) or smem (ss).
// One CTA per SM, one elected thread issues N_ITER MMAs back to back.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_24290_b200/csrc/tc_util.cuh"
using namespace rxgs_b200;

template <int N, bool TS>
__global__ void k(int iters, long long* out) {
    __shared__ __align__(1024) uint8_t sA[128 * 16 * 2];
    __shared__ __align__(1024) uint8_t sB[256 * 16 * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 16; i += blockDim.x) reinterpret_cast<uint16_t*>(sA)[i] = 0x3f80;
    for (int i = tid; i < 256 * 16; i += blockDim.x) reinterpret_cast<uint16_t*>(sB)[i] = 0x3f80;
    if (tid < 32) { tc::tmem_alloc(&tb, 512); tc::tmem_relinquish(); }
    if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t idesc = tc::idesc_bf16_f32(128, N);
    const uint64_t ad = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sA), 128, 256);
    const uint64_t bd = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sB), 128, 256);
    long long t0 = clock64();
    if (tid == 0) {
        for (int i = 0; i < iters; ++i) {
            if (TS) tc::mma_ts(tb, tb + 256, bd, idesc, 1u);
            else tc::mma_ss(tb, ad, bd, idesc, 1u);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    tc::fence_before_sync();
    __syncthreads();
    if (tid < 32) tc::tmem_dealloc(tb, 512);
}

template <int N, bool TS>
void run(const char* name) {
    long long* d; cudaMalloc(&d, 148 * 8);
    const int iters = 4096;
    k<N, TS><<<148, 128>>>(iters, d);
    cudaDeviceSynchronize();
    k<N, TS><<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    const double macs = 128.0 * N * 16;
    printf("%-12s %s  %.1f clk/MMA  %.0f MAC/clk/SM\n", name, cudaGetErrorString(e), avg / iters, macs * iters / avg);
    cudaFree(d);
}

int main() {
    run<64, true>("N64 ts");
    run<64, false>("N64 ss");
    run<128, true>("N128 ts");
    run<128, false>("N128 ss");
    run<256, true>("N256 ts");
    run<256, false>("N256 ss");
    run<16, true>("N16 ts");
    return 0;
}
