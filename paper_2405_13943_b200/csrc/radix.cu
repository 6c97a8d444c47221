// Hand-written stable LSD radix sort, onesweep style: the kernel that
// produces the keys also builds every digit's histogram, then one kernel per
// 8-bit digit ranks a 1024-4096-key tile in shared memory (warp match-any
// multisplit, stable), resolves
// its global digit offsets by decoupled look-back over earlier tiles, and
// scatters through shared memory so global writes are digit-contiguous.
// Traffic per pass: read key+value, write key+value.
#include "bsg_internal.cuh"

#include <algorithm>

namespace bsg {
namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr uint32_t kStAgg = 1u << 30, kStInc = 2u << 30, kStMask = (1u << 30) - 1;

template <typename K, int kRsItems>
__global__ __launch_bounds__(kRsThreads) void onesweep_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                              K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                              uint32_t n, int shift,
                                                              const uint32_t* __restrict__ pass_hist,
                                                              unsigned long long* status, Lookback lb) {
    pdl_prologue();
    constexpr int kRsTile = kRsThreads * kRsItems;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s_keys = reinterpret_cast<K*>(smem_raw);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * kRsTile);
    __shared__ uint32_t s_whist[kRsWarps][256];
    __shared__ uint32_t s_start[256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_scan[kRsWarps];
    __shared__ uint32_t s_gscan[kRsWarps];
    __shared__ uint32_t s_tile;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = static_cast<uint32_t>(atomicAdd(lb.ticket, 1ull) - lb.base);
    for (int i = threadIdx.x; i < kRsWarps * 256; i += kRsThreads) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t tile_base = static_cast<uint64_t>(tile) * kRsTile;

    // Warp-striped load: within a warp, item j of lane l is key w*512 + j*32 + l,
    // so processing j in order and ranking lanes in order is the input order.
    K k[kRsItems];
    uint32_t val[kRsItems];
    uint32_t rank[kRsItems];
    uint32_t dig[kRsItems];
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
        const uint64_t i = tile_base + static_cast<uint64_t>(warp) * (32 * kRsItems) + j * 32 + lane;
        if (i < n) {
            k[j] = kin[i];
            val[j] = vin[i];
            dig[j] = static_cast<uint32_t>(k[j] >> shift) & 0xffu;
        } else {
            k[j] = 0;
            val[j] = 0;
            dig[j] = 256u;  // never matches a real digit
        }
    }
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
        const unsigned peers = __match_any_sync(0xffffffffu, dig[j]);
        uint32_t base = 0;
        if (dig[j] < 256u) base = s_whist[warp][dig[j]];
        rank[j] = base + __popc(peers & lt_mask);
        __syncwarp();
        if (dig[j] < 256u && (__ffs(peers) - 1) == lane) s_whist[warp][dig[j]] = base + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // Per digit (thread = digit): exclusive prefix over warps, tile count.
    const int d = threadIdx.x;
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
        const uint32_t c = s_whist[w][d];
        s_whist[w][d] = cnt;
        cnt += c;
    }
    // Publish this tile's count, then look back for the global prefix. Status
    // word: [epoch 32 | flag 2 | count 30]; other launches' words read as unset.
    const unsigned long long tag = static_cast<unsigned long long>(lb.epoch) << 32;
    volatile unsigned long long* st = status;
    if (tile == 0) {
        atomicExch(&status[d], tag | kStInc | cnt);
    } else {
        atomicExch(&status[static_cast<uint64_t>(tile) * 256 + d], tag | kStAgg | cnt);
    }
    // Block-local exclusive scans over digits: this tile's counts (for the
    // shared-memory scatter) and the pass histogram (global digit offsets).
    const uint32_t hcnt = pass_hist[d];
    {
        uint32_t inc = cnt, ginc = hcnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            const uint32_t gy = __shfl_up_sync(0xffffffffu, ginc, o);
            if (lane >= o) {
                inc += y;
                ginc += gy;
            }
        }
        if (lane == 31) {
            s_scan[warp] = inc;
            s_gscan[warp] = ginc;
        }
        __syncthreads();
        uint32_t wp = 0, gwp = 0;
        for (int w = 0; w < warp; ++w) {
            wp += s_scan[w];
            gwp += s_gscan[w];
        }
        s_start[d] = wp + inc - cnt;
        s_base[d] = gwp + ginc - hcnt;
    }
    uint32_t prefix = 0;
    if (tile > 0) {
        int64_t p = static_cast<int64_t>(tile) - 1;
        while (p >= 0) {
            unsigned long long s;
            do {
                s = st[static_cast<uint64_t>(p) * 256 + d];
            } while ((s >> 32) != lb.epoch || (s & ~static_cast<unsigned long long>(kStMask) & 0xffffffffull) == 0);
            prefix += static_cast<uint32_t>(s) & kStMask;
            if (s & kStInc) break;
            --p;
        }
        atomicExch(&status[static_cast<uint64_t>(tile) * 256 + d], tag | kStInc | (prefix + cnt));
    }
    s_base[d] += prefix;
    __syncthreads();

#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
        if (dig[j] < 256u) {
            const uint32_t pos = s_start[dig[j]] + s_whist[warp][dig[j]] + rank[j];
            s_keys[pos] = k[j];
            s_vals[pos] = val[j];
        }
    }
    __syncthreads();
    const uint64_t rem = static_cast<uint64_t>(n) - tile_base;
    const uint32_t valid = rem < static_cast<uint64_t>(kRsTile) ? static_cast<uint32_t>(rem) : static_cast<uint32_t>(kRsTile);
    for (uint32_t i = threadIdx.x; i < valid; i += kRsThreads) {
        const K key = s_keys[i];
        const uint32_t dd = static_cast<uint32_t>(key >> shift) & 0xffu;
        const uint32_t out = s_base[dd] + (i - s_start[dd]);
        kout[out] = key;
        vout[out] = s_vals[i];
    }
}

// Digit histograms of the 8-bit digits of the V compacted 32-bit depth keys
// (V and the key width read from the step counters): shared-memory counts
// per CTA, one global atomic per non-empty bin.
__global__ __launch_bounds__(256) void depth_hist_kernel(const uint32_t* __restrict__ keys,
                                                         StepCounters* __restrict__ cnt) {
    pdl_prologue();
    __shared__ uint32_t s_h[4 * 256];
    const uint32_t n = cnt->visible;
    const int passes = depth_key_bits(cnt->visible_pre) / 8;
    uint32_t* hist = &cnt->depth_hist[0][0];
    for (int k = threadIdx.x; k < passes * 256; k += blockDim.x) s_h[k] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t key = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p * 256 + ((key >> (8 * p)) & 0xffu)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < passes * 256; k += blockDim.x)
        if (s_h[k]) atomicAdd(&hist[k], s_h[k]);
}

template <typename K, int ITEMS>
void launch_passes(Ctx* c, K* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes, uint32_t* d_hist,
                   const uint32_t* h_hist, int* sel) {
    constexpr int kTileKeys = kRsThreads * ITEMS;
    const uint32_t tiles = (n + kTileKeys - 1) / kTileKeys;
    const size_t need = static_cast<size_t>(tiles) * 256;
    if (c->radix_status_cap < need) {
        if (c->radix_status) cudaFree(c->radix_status);
        BSG_CUDA(cudaMalloc(&c->radix_status, 2 * need * sizeof(unsigned long long)));
        BSG_CUDA(cudaMemsetAsync(c->radix_status, 0, 2 * need * sizeof(unsigned long long), c->stream));  // epoch 0 is never used
        c->radix_status_cap = 2 * need;
    }
    const size_t smem = (sizeof(K) + sizeof(uint32_t)) * kTileKeys;
    BSG_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int cur = 0;
    for (int p = first_pass; p < passes; ++p) {
        if (h_hist) {
            bool trivial = false;
            for (int d = 0; d < 256; ++d)
                if (h_hist[p * 256 + d] == n) trivial = true;
            if (trivial) continue;
        }
        const Lookback lb = next_lookback(c, 1, tiles);
        launch_pdl(c->stream, tiles, kRsThreads, smem, onesweep_kernel<K, ITEMS>, keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, 8 * p, d_hist + p * 256, c->radix_status, lb);
        BSG_LAUNCHED(c);
        cur ^= 1;
    }
    *sel = cur;
}

template <typename K>
void radix_sort(Ctx* c, K* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes, uint32_t* d_hist,
                const uint32_t* h_hist, int* sel) {
    *sel = 0;
    if (n <= 1) return;
    if (n >= (1u << 30)) throw Error{BSG_ERR_CAPACITY, "radix sort supports < 2^30 keys"};
    // Tile size: the passes are look-back-latency bound at the sizes of a step
    // (V ~ 2e5 keys, P ~ 4e5 pairs). Measured at cfg 2: 2k-key tiles beat 1k
    // (depth sort 79 -> 71 us, tile sort 52 -> 43 us); 4k beat 2k from ~4e5
    // keys on (tile sort 34.5 -> 32.3 us) but not at 2e5 (depth 42 -> 46 us);
    // tiny inputs keep 1k-key tiles for SM coverage.
    if (n < (1u << 16))
        launch_passes<K, 4>(c, keys, vals, n, first_pass, passes, d_hist, h_hist, sel);
    else if (n < (1u << 18))
        launch_passes<K, 8>(c, keys, vals, n, first_pass, passes, d_hist, h_hist, sel);
    else
        launch_passes<K, 16>(c, keys, vals, n, first_pass, passes, d_hist, h_hist, sel);
}

// After a stable sort on the 32-bit range-normalised depth key (bits(z) -
// bits(zmin)) >> shift, splats whose depths fall in one key bucket (within
// 2^shift ulps) are still in row order; sort each such run by the full FP64
// depth bits, stably, so the result is the (depth, index) order of
// renderer.cpp:86-89. Runs longer than 64 (many equal keys that are not all
// equal depths) are flagged and the caller falls back to the full 64-bit sort.
__global__ void depth_tie_fixup_kernel(uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
                                       const uint64_t* __restrict__ depth_bits, uint32_t V,
                                       uint32_t* __restrict__ long_run) {
    pdl_prologue();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    const uint32_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) return;       // not a run start
    if (i + 1 >= V || keys[i + 1] != k) return;  // singleton
    uint32_t e = i + 2;
    while (e < V && keys[e] == k && e - i <= 64) ++e;
    // insertion sort by full depth; already-ordered runs (equal depths, index
    // order) cost one comparison per element, whatever their length
    uint64_t prev = depth_bits[rows[i]];
    bool sorted = true;
    for (uint32_t a = i + 1; a < e; ++a) {
        const uint64_t d = depth_bits[rows[a]];
        if (d < prev) sorted = false;
        prev = d;
    }
    if (sorted) {
        // a long run of equal keys that is already in order needs no fall-back
        if (e - i > 64) {
            uint32_t f = e;
            while (f < V && keys[f] == k) {
                const uint64_t d = depth_bits[rows[f]];
                if (d < prev) {
                    atomicOr(long_run, 1u);
                    return;
                }
                prev = d;
                ++f;
            }
        }
        return;
    }
    if (e - i > 64) {
        atomicOr(long_run, 1u);
        return;
    }
    for (uint32_t a = i + 1; a < e; ++a) {
        const uint32_t r = rows[a];
        const uint64_t d = depth_bits[r];
        uint32_t b = a;
        while (b > i && depth_bits[rows[b - 1]] > d) {
            rows[b] = rows[b - 1];
            --b;
        }
        rows[b] = r;
    }
}

}  // namespace

void radix_sort_u64(Ctx* c, uint64_t* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes,
                    uint32_t* d_hist, const uint32_t* h_hist, int* sel) {
    radix_sort<uint64_t>(c, keys, vals, n, first_pass, passes, d_hist, h_hist, sel);
}

void radix_sort_u32(Ctx* c, uint32_t* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes,
                    uint32_t* d_hist, const uint32_t* h_hist, int* sel) {
    radix_sort<uint32_t>(c, keys, vals, n, first_pass, passes, d_hist, h_hist, sel);
}

void launch_depth_hist(Ctx* c, const uint32_t* keys) {
    const unsigned grid = std::min<unsigned>(static_cast<unsigned>((c->n + 4095) / 4096), 148);  // upper bound V <= n
    launch_pdl(c->stream, std::max(grid, 1u), 256, 0, depth_hist_kernel, keys, c->counters);
    BSG_LAUNCHED(c);
}

void depth_tie_fixup(Ctx* c, uint32_t* keys, uint32_t* rows, const uint64_t* depth_bits, uint32_t V,
                     uint32_t* long_run) {
    if (V < 2) return;
    launch_pdl(c->stream, (V + 255) / 256, 256, 0, depth_tie_fixup_kernel, keys, rows, depth_bits, V, long_run);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
