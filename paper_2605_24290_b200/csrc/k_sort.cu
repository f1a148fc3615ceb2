// Tile binning: the device form of bin_and_sort (sphraster.cpp:85-102).
//
// The reference pushes Gaussian indices into each covered tile in index
// order and std::stable_sort's every list by FP64 depth, i.e. each list is
// ordered by (depth, index).  On the device:
//   1. radix-sort all K Gaussians by the IEEE bits of their FP64 depth
//      (positive doubles order like their bit patterns; culled -> ~0).  The
//      sort is stable over an index-ordered input, so ties keep index order:
//      rank[g] = position of g in (depth, index) order;
//   2. scan the per-Gaussian tile counts in rank order and emit one
//      (tile, g) pair per covered tile, in rank order;
//   3. stable radix sort of the pairs by the tile id alone (ceil(log2 tiles)
//      bits, 2 passes at 12 bits): within a tile the rank order survives;
//   4. per-tile [begin, end) from the tile-id steps of the sorted pairs, and the 64-bit sort keys
//      (tile << 32) | rank that the north star asks to be bit-exact.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

__global__ void k_iota(int n, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__global__ void k_rank(int K, const int* __restrict__ order, const int* __restrict__ tile_count,
                       const uint64_t* __restrict__ depth_key, int* __restrict__ rank,
                       int64_t* __restrict__ cnt_sorted, unsigned long long* __restrict__ n_culled) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > K) return;
    if (r == K) {
        cnt_sorted[K] = 0;
        return;
    }
    const int g = order[r];
    rank[g] = r;
    cnt_sorted[r] = tile_count[g];
    if (depth_key[g] == ~0ull) atomicAdd(n_culled, 1ull);
}

__global__ void k_emit(int K, int tiles_p, const int* __restrict__ order,
                       const int4* __restrict__ spans, const int64_t* __restrict__ scan,
                       uint32_t* __restrict__ tkey, int* __restrict__ tval) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= K) return;
    const int64_t begin = scan[r];
    const int64_t n = scan[r + 1] - begin;
    if (n == 0) return;
    const int g = order[r];
    const int4 sp = spans[g];
    int64_t o = begin;
    for (int tt = sp.x; tt <= sp.y; ++tt)
        for (int pp = sp.z; pp <= sp.w; ++pp) {
            const int tile = tt * tiles_p + pp % tiles_p;
            tkey[o] = static_cast<uint32_t>(tile);
            tval[o] = g;
            ++o;
        }
}

__global__ void k_keys(int64_t n, const uint32_t* __restrict__ tkey, const int* __restrict__ list,
                       const int* __restrict__ rank, uint64_t* __restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    keys[i] = (static_cast<uint64_t>(tkey[i]) << 32) | static_cast<uint32_t>(rank[list[i]]);
}

// tile_offsets[t] = first position of tile t in the tile-sorted pairs
// (= lower_bound), written by the entry where the tile id steps up; no
// histogram atomics.
__global__ void k_offsets(int64_t n, int n_tiles, const uint32_t* __restrict__ tks, int64_t* __restrict__ off) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > n) return;
    const int prev = i == 0 ? -1 : static_cast<int>(tks[i - 1]);
    const int cur = i == n ? n_tiles : static_cast<int>(tks[i]);
    for (int t = prev + 1; t <= cur; ++t) off[t] = i;
}

int bits_for(int n) {
    int b = 1;
    while ((1 << b) < n) ++b;
    return b;
}

}  // namespace

int bin_tiles(rxgs_ctx ctx, rxgs_txstate_s& st, cudaStream_t s) {
    const int K = st.k;
    const int n_tiles = st.grid.n_tiles;
    RXGS_CUDA(st.order.ensure(sizeof(int) * (K + 1)));
    RXGS_CUDA(st.rank.ensure(sizeof(int) * (K + 1)));
    RXGS_CUDA(st.scan.ensure(sizeof(int64_t) * (K + 1)));
    RXGS_CUDA(st.tile_offsets.ensure(sizeof(int64_t) * (n_tiles + 1)));

    // scratch: sorted depth keys (K u64) | iota (K int) | cnt_sorted (K+1 i64) |
    // [total, culled] (every sub-buffer 256-byte aligned)
    auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    const size_t off_iota = al(sizeof(uint64_t) * (K + 1));
    const size_t off_cnt = off_iota + al(sizeof(int) * (K + 2));
    const size_t off_red = off_cnt + al(sizeof(int64_t) * (K + 2));
    RXGS_CUDA(ctx->scratch_a.ensure(off_red + 256));
    char* base = ctx->scratch_a.as<char>();
    uint64_t* dk_sorted = reinterpret_cast<uint64_t*>(base);
    int* iota = reinterpret_cast<int*>(base + off_iota);
    int64_t* cnt_sorted = reinterpret_cast<int64_t*>(base + off_cnt);
    int64_t* red = reinterpret_cast<int64_t*>(base + off_red);  // [0] entries, [1] culled

    RXGS_CUDA(cudaMemsetAsync(red, 0, 2 * sizeof(int64_t), s));
    if (K > 0) {
        k_iota<<<(K + 255) / 256, 256, 0, s>>>(K, iota);
        size_t tmp = 0;
        RXGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, st.depth_key.as<uint64_t>(), dk_sorted,
                                                  iota, st.order.as<int>(), K, 0, 64, s));
        RXGS_CUDA(ctx->sort_tmp.ensure(tmp));
        RXGS_CUDA(cub::DeviceRadixSort::SortPairs(ctx->sort_tmp.p, tmp, st.depth_key.as<uint64_t>(),
                                                  dk_sorted, iota, st.order.as<int>(), K, 0, 64, s));
        k_rank<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, st.order.as<int>(), st.tile_count.as<int>(),
                                                   st.depth_key.as<uint64_t>(), st.rank.as<int>(),
                                                   cnt_sorted, reinterpret_cast<unsigned long long*>(red + 1));
        tmp = 0;
        RXGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt_sorted, st.scan.as<int64_t>(), K + 1, s));
        RXGS_CUDA(ctx->sort_tmp.ensure(tmp));
        RXGS_CUDA(cub::DeviceScan::ExclusiveSum(ctx->sort_tmp.p, tmp, cnt_sorted, st.scan.as<int64_t>(),
                                                K + 1, s));
    }
    int64_t total = 0, culled = 0;
    if (K > 0) {
        RXGS_CUDA(cudaMemcpyAsync(&total, st.scan.as<int64_t>() + K, sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaMemcpyAsync(&culled, red + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaStreamSynchronize(s));
    }
    st.entries = total;
    st.visible = K - culled;
    RXGS_CUDA(st.list.ensure(sizeof(int) * (total + 1)));
    RXGS_CUDA(st.keys.ensure(sizeof(uint64_t) * (total + 1)));
    // pair scratch: tkey | tval | tkey_sorted
    const size_t o_tval = sizeof(uint32_t) * (total + 1);
    const size_t o_tks = o_tval + sizeof(int) * (total + 1);
    RXGS_CUDA(ctx->scratch_b.ensure(o_tks + sizeof(uint32_t) * (total + 1)));
    char* pb = ctx->scratch_b.as<char>();
    uint32_t* tkey = reinterpret_cast<uint32_t*>(pb);
    int* tval = reinterpret_cast<int*>(pb + o_tval);
    uint32_t* tks = reinterpret_cast<uint32_t*>(pb + o_tks);
    if (total > 0) {
        k_emit<<<(K + 127) / 128, 128, 0, s>>>(K, st.grid.tiles_p, st.order.as<int>(), st.spans.as<int4>(),
                                               st.scan.as<int64_t>(), tkey, tval);
        size_t tmp = 0;
        const int end_bit = bits_for(n_tiles);
        RXGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, tkey, tks, tval, st.list.as<int>(),
                                                  static_cast<int>(total), 0, end_bit, s));
        RXGS_CUDA(ctx->sort_tmp.ensure(tmp));
        RXGS_CUDA(cub::DeviceRadixSort::SortPairs(ctx->sort_tmp.p, tmp, tkey, tks, tval,
                                                  st.list.as<int>(), static_cast<int>(total), 0,
                                                  end_bit, s));
        k_keys<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(total, tks, st.list.as<int>(),
                                                                          st.rank.as<int>(),
                                                                          st.keys.as<uint64_t>());
    }
    k_offsets<<<static_cast<unsigned>((total + 1 + 255) / 256), 256, 0, s>>>(total, n_tiles, tks,
                                                                              st.tile_offsets.as<int64_t>());
    ctx->launches += 8;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "bin_tiles");
}

}  // namespace rxgs_b200

// ---------------------------------------------------------------- needed rows
#include <cub/device/device_select.cuh>

namespace rxgs_b200 {
namespace {

__global__ void k_mark_needed(DevGrid g, const int64_t* __restrict__ tile_offsets, const int* __restrict__ list,
                              const int* __restrict__ walk_len, unsigned char* __restrict__ needed) {
    const int tile = blockIdx.x;
    int w = 0;
    for (int b = 0; b < g.cell_blocks; ++b) w = max(w, walk_len[tile * g.cell_blocks + b]);
    const int64_t begin = tile_offsets[tile];
    for (int p = threadIdx.x; p < w; p += blockDim.x) needed[list[begin + p]] = 1;
}

__global__ void k_flags_in_order(int n, const int* __restrict__ order, const unsigned char* __restrict__ needed,
                                 unsigned char* __restrict__ flags) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) flags[r] = needed[order[r]];
}

}  // namespace

int compact_needed(rxgs_ctx ctx, const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s) {
    const int K = st.k;
    RXGS_CUDA(st.needed.ensure(static_cast<size_t>(K + 1) * 2));
    RXGS_CUDA(st.needed_order.ensure(sizeof(int) * (K + 1)));
    RXGS_CUDA(st.needed_count.ensure(sizeof(int) * 4));
    unsigned char* needed = st.needed.as<unsigned char>();
    unsigned char* flags = needed + (K + 1);
    RXGS_CUDA(cudaMemsetAsync(needed, 0, static_cast<size_t>(K + 1), s));
    RXGS_CUDA(cudaMemsetAsync(st.needed_count.p, 0, sizeof(int), s));
    if (st.entries > 0)
        k_mark_needed<<<st.grid.n_tiles, 128, 0, s>>>(st.grid, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                                                       st.walk_len.as<int>(), needed);
    if (st.visible > 0 && K > 0) {
        // compact in the scene's spatial (Morton) order: consecutive
        // conditioning rows are nearby Gaussians (k_cond_tc.cu)
        k_flags_in_order<<<(K + 255) / 256, 256, 0, s>>>(K, sc.d_morton.as<int>(), needed, flags);
        size_t tmp = 0;
        RXGS_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, sc.d_morton.as<int>(), flags, st.needed_order.as<int>(),
                                             st.needed_count.as<int>(), K, s));
        RXGS_CUDA(ctx->sort_tmp.ensure(tmp));
        RXGS_CUDA(cub::DeviceSelect::Flagged(ctx->sort_tmp.p, tmp, sc.d_morton.as<int>(), flags,
                                             st.needed_order.as<int>(), st.needed_count.as<int>(), K, s));
    }
    st.needed_host = -1;
    if (ctx->profile) {  // roofline bookkeeping only: the row count of the next conditioning launch
        int h = 0;
        RXGS_CUDA(cudaMemcpyAsync(&h, st.needed_count.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaStreamSynchronize(s));
        st.needed_host = h;
    }
    ctx->launches += 3;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "compact_needed");
}

// ------------------------------------------------------------- scene order
// Morton (Z-order) permutation of the scene's Gaussians over their bounding
// box, 10 bits per axis: the spatial order the conditioning kernel walks
// rows in, so a warp's 32 occupancy probes stay within a few voxels.
namespace {
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__global__ void k_morton(int K, const float4* __restrict__ pos, float lx, float ly, float lz, float sx, float sy,
                         float sz, uint32_t* __restrict__ key, int* __restrict__ idx) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const float4 p = pos[k];
    auto q = [](float v, float lo, float sc) {
        const float u = (v - lo) * sc;
        return static_cast<uint32_t>(fminf(fmaxf(u, 0.f), 1023.f));
    };
    key[k] = (spread3(q(p.x, lx, sx)) << 2) | (spread3(q(p.y, ly, sy)) << 1) | spread3(q(p.z, lz, sz));
    idx[k] = k;
}
__global__ void k_gather_pos(int K, const int* __restrict__ order, const float4* __restrict__ pos,
                             float4* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < K) out[r] = pos[order[r]];
}
}  // namespace

int build_scene_order(rxgs_ctx ctx, rxgs_scene_s& sc, cudaStream_t s) {
    const int K = sc.k;
    RXGS_CUDA(sc.d_morton.ensure(sizeof(int) * std::max(K, 1)));
    RXGS_CUDA(sc.d_mpos32.ensure(sizeof(float4) * std::max(K, 1)));
    if (K == 0) return RXGS_OK;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = 1.7976931348623157e308;
        hi[a] = -1.7976931348623157e308;
    }
    for (int k = 0; k < K; ++k)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], sc.h_pos[3 * k + a]);
            hi[a] = std::max(hi[a], sc.h_pos[3 * k + a]);
        }
    float scale[3];
    for (int a = 0; a < 3; ++a) scale[a] = hi[a] > lo[a] ? static_cast<float>(1024.0 / (hi[a] - lo[a])) : 0.f;
    DevBuf keys;
    RXGS_CUDA(keys.ensure(static_cast<size_t>(K) * 2 * (sizeof(uint32_t) + sizeof(int))));
    uint32_t* k_in = keys.as<uint32_t>();
    uint32_t* k_out = k_in + K;
    int* i_in = reinterpret_cast<int*>(k_out + K);
    k_morton<<<(K + 255) / 256, 256, 0, s>>>(K, sc.d_pos32.as<float4>(), static_cast<float>(lo[0]),
                                              static_cast<float>(lo[1]), static_cast<float>(lo[2]), scale[0],
                                              scale[1], scale[2], k_in, i_in);
    size_t tmp = 0;
    RXGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k_in, k_out, i_in, sc.d_morton.as<int>(), K, 0, 30, s));
    RXGS_CUDA(ctx->sort_tmp.ensure(tmp));
    RXGS_CUDA(cub::DeviceRadixSort::SortPairs(ctx->sort_tmp.p, tmp, k_in, k_out, i_in, sc.d_morton.as<int>(), K, 0,
                                              30, s));
    k_gather_pos<<<(K + 255) / 256, 256, 0, s>>>(K, sc.d_morton.as<int>(), sc.d_pos32.as<float4>(),
                                                  sc.d_mpos32.as<float4>());
    RXGS_CUDA(cudaStreamSynchronize(s));  // keys is freed on return
    return RXGS_OK;
}

}  // namespace rxgs_b200
