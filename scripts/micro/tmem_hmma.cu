// Microbenchmarks for the conditioning kernel's design choice (one CTA per SM):
//  (1) tcgen05.ld throughput (32x32b.x16/.x32/.x64) with W warps per CTA;
//  (2) legacy mma.sync.m16n8k16 bf16 -> f32 throughput with W warps per CTA;
//  (3) FFMA2 issue throughput for reference.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_24290_b200/csrc/tc_util.cuh"
using namespace rxgs_b200;

template <int X>
__device__ __forceinline__ uint32_t ldx(uint32_t taddr);
template <>
__device__ __forceinline__ uint32_t ldx<16>(uint32_t taddr) {
    uint32_t r[16];
    tc::tmem_ld16(taddr, r);
    tc::wait_ld_regs(r);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= r[i];
    return x;
}
template <>
__device__ __forceinline__ uint32_t ldx<32>(uint32_t taddr) {
    uint32_t r[16], s[16];
    tc::tmem_ld16(taddr, r);
    tc::tmem_ld16(taddr + 16, s);
    tc::wait_ld_regs(r);
    tc::wait_ld_regs(s);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= r[i] ^ s[i];
    return x;
}
template <>
__device__ __forceinline__ uint32_t ldx<64>(uint32_t taddr) {
    uint32_t r[16], s[16], t[16], u[16];
    tc::tmem_ld16(taddr, r);
    tc::tmem_ld16(taddr + 16, s);
    tc::tmem_ld16(taddr + 32, t);
    tc::tmem_ld16(taddr + 48, u);
    tc::wait_ld_regs(r);
    tc::wait_ld_regs(s);
    tc::wait_ld_regs(t);
    tc::wait_ld_regs(u);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= r[i] ^ s[i] ^ t[i] ^ u[i];
    return x;
}

template <int X>
__global__ void k_tmem(int iters, long long* cyc, uint32_t* sink) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc::tmem_alloc(&tb, 512); tc::tmem_relinquish(); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t base = tb + ((static_cast<uint32_t>(32 * (warp & 3))) << 16) + 64 * ((warp >> 2) & 7);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) acc ^= ldx<X>(base + (i & 1) * 0);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tb, 512);
}

__global__ void k_hmma(int iters, long long* cyc, float* sink) {
    uint32_t a0 = 0x3f803f80u + threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = 0x3f803f80u, b1 = b0 ^ 5;
    float d[4][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(d[q][0]), "+f"(d[q][1]), "+f"(d[q][2]), "+f"(d[q][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
    for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
    if (s == 1234.5f) sink[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, sizeof(long long) * sms);
    cudaMalloc(&sink, 64);
    long long h[256];
    const int iters = 4096;
    auto run_tmem = [&](auto kern, int X, int warps) {
        kern<<<sms, 32 * warps>>>(iters, cyc, sink);
        kern<<<sms, 32 * warps>>>(iters, cyc, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double c = 0;
        for (int i = 0; i < sms; ++i) c += h[i];
        c /= sms;
        const double bytes = static_cast<double>(warps) * iters * 32 * X * 4;
        printf("tcgen05.ld 32x32b x%d  warps %2d : %.1f B/clk/SM  (%.0f clk)  err=%s\n", X, warps, bytes / c, c,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int w : {4, 8, 16, 32}) {
        run_tmem(k_tmem<16>, 16, w);
        run_tmem(k_tmem<32>, 32, w);
        run_tmem(k_tmem<64>, 64, w);
    }
    for (int w : {4, 8, 16, 32}) {
        k_hmma<<<sms, 32 * w>>>(iters, cyc, reinterpret_cast<float*>(sink));
        k_hmma<<<sms, 32 * w>>>(iters, cyc, reinterpret_cast<float*>(sink));
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double c = 0;
        for (int i = 0; i < sms; ++i) c += h[i];
        c /= sms;
        const double macs = static_cast<double>(w) * iters * 4 * 16 * 8 * 16;
        printf("mma.sync m16n8k16 bf16 warps %2d : %.0f MAC/clk/SM (%s)\n", w, macs / c,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
