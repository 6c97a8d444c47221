// K3-K8: tile pairs, tile ranges, forward blend and reverse-traversal
// backward blend. Replaces bin_splats and the per-pixel compositing loops of
// render / render_backward (renderer.cpp:99-117,150-183,236-311).
//
// The reference bins every splat into every pixel of its integer footprint
// rect. Here a splat is duplicated into every 16x16 tile its rect overlaps,
// pairs are emitted in (depth, index) order and stably sorted by tile, and
// each pixel re-applies the exact rect test while walking its tile's list, so
// a pixel sees exactly the reference's contributor list in the reference's
// order. Blending is FP32 (exp through MUFU).
#include "bsg_internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace bsg {
namespace {

__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void unpack_rect(const float4& c, int& x0, int& x1, int& y0, int& y1) {
    const uint32_t r01 = __float_as_uint(c.y), r23 = __float_as_uint(c.z);
    x0 = static_cast<int>(r01 & 0xffffu);
    x1 = static_cast<int>(r01 >> 16);
    y0 = static_cast<int>(r23 & 0xffffu);
    y1 = static_cast<int>(r23 >> 16);
}

// One thread per depth-sorted splat: write (tile, row) for every overlapped tile.
__global__ __launch_bounds__(256) void emit_pairs_kernel(const uint32_t* __restrict__ sorted_rows,
                                                         const uint32_t* __restrict__ offsets,
                                                         const float4* __restrict__ rec, uint32_t V, int tiles_x,
                                                         uint32_t* __restrict__ pkey, uint32_t* __restrict__ pval,
                                                         uint32_t pcap, uint32_t* __restrict__ hist,
                                                         uint2* __restrict__ ranges, uint32_t ntiles) {
    pdl_prologue();
    __shared__ uint32_t s_hist[2 * 256];
    for (int k = threadIdx.x; k < 512; k += blockDim.x) s_hist[k] = 0;
    // tiles without pairs keep the empty range (ranges_kernel writes the rest)
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
        ranges[t] = make_uint2(0u, 0u);
    __syncthreads();
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < V) {
        const uint32_t row = sorted_rows[p];
        int x0, x1, y0, y1;
        unpack_rect(rec[3 * static_cast<size_t>(row) + 2], x0, x1, y0, y1);
        uint32_t o = offsets[p];
        for (int ty = y0 / kTile; ty <= y1 / kTile; ++ty)
            for (int tx = x0 / kTile; tx <= x1 / kTile; ++tx) {
                const uint32_t key = static_cast<uint32_t>(ty * tiles_x + tx);
                if (o < pcap) {
                    pkey[o] = key;
                    pval[o] = row;
                }
                atomicAdd(&s_hist[key & 0xffu], 1u);
                atomicAdd(&s_hist[256 + ((key >> 8) & 0xffu)], 1u);
                ++o;
            }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 512; k += blockDim.x)
        if (s_hist[k]) atomicAdd(&hist[k], s_hist[k]);
}

__global__ __launch_bounds__(256) void ranges_kernel(const uint32_t* __restrict__ pkey, uint32_t P,
                                                     uint2* __restrict__ ranges) {
    pdl_prologue();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t k = pkey[i];
    if (i == 0 || pkey[i - 1] != k) ranges[k].x = i;
    if (i == P - 1 || pkey[i + 1] != k) ranges[k].y = i + 1;
}

// ---- per-tile binning (the default path) --------------------------------
// The preprocess counts each visible splat into every tile its rect overlaps.
// K4a scans the counts into tile ranges and emission cursors (one CTA), and
// publishes P and the largest tile count; K4b places every visible splat's row
// into each of its tiles at an atomically claimed slot (order inside a tile is
// arbitrary); K5 sorts each tile's rows in shared memory by (FP64 depth bits,
// row) -- exactly the reference's stable (depth, index) order restricted to
// the tile (renderer.cpp:86-89) -- replacing the global depth sort, its tie
// fix-up and the stable tile-key sort.

// One CTA: exclusive scan of the tile counts -> ranges and cursors, the blend
// launch order (descending count), and P / max count to the mailbox. The
// tiles are walked in chunks of 1024 (tile = chunk base + thread), so every
// load and store is coalesced; each chunk is block-scanned with a running
// carry. (A thread-per-7-consecutive-tiles layout made every access a
// 28-byte-strided gather: 47 us at cfg 3's 6700 tiles.)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t ex = (warp ? s_warp[warp - 1] : 0u) + inc - v;
    total = s_warp[31];
    __syncthreads();
    return ex;
}

__global__ __launch_bounds__(1024) void tile_scan_kernel(const uint32_t* __restrict__ cnt, uint32_t ntiles,
                                                         uint2* __restrict__ ranges, uint32_t* __restrict__ cur,
                                                         uint32_t* __restrict__ order, Mailbox* mb, uint32_t seq,
                                                         uint32_t* __restrict__ pairs_dev) {
    pdl_prologue();
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_bucket[1024];
    __shared__ uint32_t s_max;
    __shared__ unsigned long long s_total;  // P without 32-bit wrap-around (the capacity guard)
    const uint32_t t = threadIdx.x;
    s_bucket[t] = 0;
    if (t == 0) {
        s_max = 0;
        s_total = 0;
    }
    __syncthreads();
    // ranges, cursors and the launch-order histogram (bucket 1023 - min(count, 1023))
    uint32_t carry = 0, mx = 0;
    unsigned long long wide = 0;
    static_assert(kTileSub == 4, "one uint4 of sub-counts per tile");
    const uint4* cnt4 = reinterpret_cast<const uint4*>(cnt);
    uint4* cur4 = reinterpret_cast<uint4*>(cur);
    for (uint32_t c0 = 0; c0 < ntiles; c0 += 1024) {
        const uint32_t i = c0 + t;
        const uint4 sc = i < ntiles ? cnt4[i] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t v = sc.x + sc.y + sc.z + sc.w;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, s_warp, total);
        if (i < ntiles) {
            const uint32_t b = carry + ex;
            ranges[i] = make_uint2(b, b + v);
            cur4[i] = make_uint4(b, b + sc.x, b + sc.x + sc.y, b + sc.x + sc.y + sc.z);  // sub-ranges end to end
            atomicAdd(&s_bucket[1023u - min(v, 1023u)], 1u);
        }
        carry += total;
        mx = max(mx, v);
        wide += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        wide += __shfl_xor_sync(0xffffffffu, wide, o);
    }
    if ((t & 31) == 0) {
        atomicMax(&s_max, mx);
        atomicAdd(&s_total, wide);
    }
    __syncthreads();
    // bucket offsets (exclusive scan of the 1024 bucket counts)
    {
        uint32_t total;
        const uint32_t b = s_bucket[t];
        const uint32_t ex = block_exclusive_scan(b, s_warp, total);
        s_bucket[t] = ex;
        __syncthreads();
    }
    // launch order: tiles by descending count (order inside a bucket is free)
    for (uint32_t c0 = 0; c0 < ntiles; c0 += 1024) {
        const uint32_t i = c0 + t;
        if (i < ntiles) {
            const uint4 sc = cnt4[i];
            order[atomicAdd(&s_bucket[1023u - min(sc.x + sc.y + sc.z + sc.w, 1023u)], 1u)] = i;
        }
    }
    if (t == 0) {
        *pairs_dev = carry;
        *reinterpret_cast<volatile uint32_t*>(&mb->P) = carry;
        *reinterpret_cast<volatile uint32_t*>(&mb->max_tile) = s_max;
        *reinterpret_cast<volatile uint32_t*>(&mb->pairs_big) = s_total >= kMaxPairs ? 1u : 0u;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&mb->seq_p) = seq;
    }
}

// One thread per visible splat (grid-stride; V from the step counters): its
// row into every tile it overlaps, at a slot claimed from the tile's cursor.
__global__ __launch_bounds__(256) void emit_tiles_kernel(const uint32_t* __restrict__ vis_rows,
                                                         const StepCounters* __restrict__ counters,
                                                         const float4* __restrict__ rec, int tiles_x,
                                                         uint32_t* __restrict__ cur, uint32_t* __restrict__ out_rows,
                                                         uint32_t pcap, const uint2* __restrict__ ranges_end) {
    pdl_prologue();
    const uint32_t V = counters->visible;
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < V; p += gridDim.x * blockDim.x) {
        const uint32_t row = vis_rows[p];
        int x0, x1, y0, y1;
        unpack_rect(rec[3 * static_cast<size_t>(row) + 2], x0, x1, y0, y1);
        // the row's slot claims are independent: up to 4 in flight at once
        // (the kernel is bound by the claims' L2 round trips)
        const int tx0 = x0 / kTile, ty0 = y0 / kTile, w = x1 / kTile - tx0 + 1;
        const int nt = w * (y1 / kTile - ty0 + 1);
        for (int b = 0; b < nt; b += 4) {
            uint32_t slot[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (b + k < nt) {
                    const int ty = ty0 + (b + k) / w, tx = tx0 + (b + k) % w;
                    slot[k] = atomicAdd(&cur[kTileSub * (ty * tiles_x + tx) + (row & (kTileSub - 1))], 1u);
                    BSG_DASSERT(slot[k] < ranges_end[ty * tiles_x + tx].y);  // the tile's cursor stays in its range
                }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (b + k < nt && slot[k] < pcap) out_rows[slot[k]] = row;
        }
    }
}

constexpr int kTieRounds = 32;  // odd-even rounds before the full-key re-sort (runs can be ~2048 long)
constexpr uint32_t kTileSortThreads = 128;

// Bitonic sort of a tile's N <= EPT x kTileSortThreads packed keys in
// registers, EPT consecutive positions per thread: a stage's partner is in the
// same thread (distance < EPT), a lane of the same warp (distance < 32 EPT:
// shuffles) or another warp (through shared memory). The sorted keys end in sk.
// (cfg 3 sort stage: shared-memory network 58.7 us, registers up to 256 pairs
// 51.0, up to 1024 pairs 49.5.)
template <int EPT>
__device__ __forceinline__ void tile_sort_regs(uint64_t* __restrict__ sk, const uint32_t* __restrict__ rows,
                                               uint32_t n, uint32_t N, const uint64_t* __restrict__ depth_key) {
    const uint32_t p0 = EPT * threadIdx.x;
    uint64_t v[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        v[e] = ~0ull;  // padding sorts last
        if (p0 + e < n) {
            const uint32_t row = rows[p0 + e];
            v[e] = (depth_key[row] & 0xffffffff00000000ull) | row;
        }
    }
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j < EPT) {
#pragma unroll
                for (int jj = EPT / 2; jj >= 1; jj >>= 1)
                    if (jj == static_cast<int>(j)) {
#pragma unroll
                        for (int e = 0; e < EPT; ++e)
                            if ((e & jj) == 0) {
                                const bool up = ((p0 + e) & k) == 0;
                                if ((v[e] > v[e | jj]) == up) {
                                    const uint64_t tmp = v[e];
                                    v[e] = v[e | jj];
                                    v[e | jj] = tmp;
                                }
                            }
                    }
                continue;
            }
            // j >= EPT: all of the thread's positions share bits j and k
            const bool keep_min = ((p0 & j) == 0) == ((p0 & k) == 0);
            uint64_t o[EPT];
            if (j < 32u * EPT) {
#pragma unroll
                for (int e = 0; e < EPT; ++e) o[e] = __shfl_xor_sync(0xffffffffu, v[e], j / EPT);
            } else {
                if (p0 < N) {
#pragma unroll
                    for (int e = 0; e < EPT; ++e) sk[p0 + e] = v[e];
                }
                __syncthreads();
#pragma unroll
                for (int e = 0; e < EPT; ++e) o[e] = p0 < N ? sk[(p0 + e) ^ j] : v[e];
                __syncthreads();
            }
#pragma unroll
            for (int e = 0; e < EPT; ++e) v[e] = keep_min ? (o[e] < v[e] ? o[e] : v[e]) : (o[e] > v[e] ? o[e] : v[e]);
        }
    }
    if (p0 < N) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) sk[p0 + e] = v[e];
    }
}

// One CTA per tile: the tile's rows sorted by (FP64 depth bits, row) with a
// bitonic network in shared memory (size: the next power of two of the
// tile's count, at most kTileSortCap; dynamic shared memory sized for the
// view's largest tile). Tiles in the blend launch order (longest first).
__global__ __launch_bounds__(kTileSortThreads) void tile_sort_kernel(const uint2* __restrict__ ranges,
                                                        const uint32_t* __restrict__ order,
                                                        const uint32_t* __restrict__ rows_in,
                                                        const uint64_t* __restrict__ depth_key,
                                                        uint32_t* __restrict__ rows_out) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint2 r = ranges[order[blockIdx.x]];  // longest tiles first
    const uint32_t n = r.y - r.x;
    if (n == 0) return;
    if (n == 1) {
        if (threadIdx.x == 0) rows_out[r.x] = rows_in[r.x];
        return;
    }
    uint32_t N = 2;
    while (N < n) N <<= 1;
    BSG_DASSERT(N <= kTileSortCap);
    // one 64-bit word per pair: the upper 32 bits of the FP64 depth (its sign,
    // exponent and 20 mantissa bits: order-preserving for positive depths) and
    // the row, so a compare-exchange moves one word; pairs whose upper depth
    // bits tie are put in (full depth, row) order afterwards
    uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
    if (N <= 2 * kTileSortThreads) {
        tile_sort_regs<2>(sk, rows_in + r.x, n, N, depth_key);
    } else if (N <= 4 * kTileSortThreads) {
        tile_sort_regs<4>(sk, rows_in + r.x, n, N, depth_key);
    } else if (N <= 8 * kTileSortThreads) {
        tile_sort_regs<8>(sk, rows_in + r.x, n, N, depth_key);
    } else {
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        if (i < n) {
            const uint32_t row = rows_in[r.x + i];
            sk[i] = (depth_key[row] & 0xffffffff00000000ull) | row;
        } else {
            sk[i] = ~0ull;  // padding sorts last
        }
    }
    __syncthreads();
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            // pairs with j <= 32 stay inside the 64 elements of one warp's
            // 32 compare-exchanges: those stages only need a warp barrier
            for (uint32_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                // i-th compare-exchange pair of this stage: a has bit j clear
                const uint32_t a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                const uint32_t b = a | j;
                const bool up = (a & k) == 0;
                const uint64_t ka = sk[a], kb = sk[b];
                if ((ka > kb) == up) {
                    sk[a] = kb;
                    sk[b] = ka;
                }
            }
            const uint32_t jn = j > 1 ? j >> 1 : k;  // the next stage's distance
            if (j >= 64 || jn >= 64)
                __syncthreads();
            else
                __syncwarp();
        }
    }
    }
    __syncthreads();
    // runs of equal upper depth bits (depths within ~1e-6 relative): odd-even
    // transposition by (full FP64 depth, row) until a round swaps nothing --
    // at most kTieRounds rounds (short runs, the common case); a tile whose
    // runs are longer is re-sorted by the full key below
    bool sorted = false;
    for (int round = 0; round < kTieRounds; ++round) {
        bool swapped = false;
        for (uint32_t parity = 0; parity < 2; ++parity) {
            for (uint32_t i = 2 * threadIdx.x + parity; i + 1 < n; i += 2 * blockDim.x) {
                const uint64_t ka = sk[i], kb = sk[i + 1];
                if ((ka >> 32) != (kb >> 32)) continue;
                const uint32_t ra = static_cast<uint32_t>(ka), rb = static_cast<uint32_t>(kb);
                const uint64_t da = depth_key[ra], db = depth_key[rb];
                if (da > db || (da == db && ra > rb)) {
                    sk[i] = kb;
                    sk[i + 1] = ka;
                    swapped = true;
                }
            }
            __syncthreads();
        }
        if (!__syncthreads_or(swapped)) {
            sorted = true;
            break;
        }
    }
    if (!sorted) {
        // long runs of near-equal depths: one bitonic network over the full
        // (FP64 depth bits, row) key, rows alongside (the shared memory holds
        // kTileSortCap x 12 B)
        uint32_t* srow = reinterpret_cast<uint32_t*>(sk + N);
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
            const uint32_t row = i < n ? static_cast<uint32_t>(sk[i]) : 0xffffffffu;
            srow[i] = row;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) sk[i] = i < n ? depth_key[srow[i]] : ~0ull;
        __syncthreads();
        for (uint32_t k = 2; k <= N; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                    const uint32_t a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                    const uint32_t b = a | j;
                    const bool up = (a & k) == 0;
                    const uint64_t ka = sk[a], kb = sk[b];
                    const uint32_t ra = srow[a], rb = srow[b];
                    if ((ka > kb || (ka == kb && ra > rb)) == up) {
                        sk[a] = kb;
                        sk[b] = ka;
                        srow[a] = rb;
                        srow[b] = ra;
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) rows_out[r.x + i] = srow[i];
        return;
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) rows_out[r.x + i] = static_cast<uint32_t>(sk[i]);
}

// Blend launch order: tiles sorted by descending pair count (longest
// processing time first), so the heaviest tiles start in the first wave and
// the light ones fill the tail of the ~2.5 waves. One CTA, counting sort on
// min(count, 1023); the order inside a bucket is free (tiles are
// independent, every output is per tile). List-scheduling model on the cfg 2
// views' tile counts: 7-19% shorter makespan than row-major order.
__global__ __launch_bounds__(1024) void tile_order_kernel(const uint2* __restrict__ ranges, uint32_t ntiles,
                                                          uint32_t* __restrict__ order) {
    pdl_prologue();
    __shared__ uint32_t s_cnt[1024];
    __shared__ uint32_t s_warp[32];
    const uint32_t t = threadIdx.x;
    s_cnt[t] = 0;
    __syncthreads();
    for (uint32_t i = t; i < ntiles; i += 1024) {
        const uint2 r = ranges[i];
        atomicAdd(&s_cnt[1023u - min(r.y - r.x, 1023u)], 1u);
    }
    __syncthreads();
    // exclusive scan of the 1024 bucket counts
    const uint32_t v = s_cnt[t];
    uint32_t inc = v;
    const int lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi - w;
    }
    __syncthreads();
    s_cnt[t] = s_warp[warp] + inc - v;
    __syncthreads();
    for (uint32_t i = t; i < ntiles; i += 1024) {
        const uint2 r = ranges[i];
        order[atomicAdd(&s_cnt[1023u - min(r.y - r.x, 1023u)], 1u)] = i;
    }
}

// K7 blend forward: one CTA of 128 threads per 16x16 tile. Warp w owns the
// 8x8 sub-tile (w & 1, w >> 1); each lane owns two pixels of it (rows ly and
// ly + 4), so every shared-memory record load serves two pixels. Splat
// records are staged 256 at a time; staging turns each record into the
// tile-local affine form of its conic (see stage_entry) and builds, per warp,
// a 16-bit hit mask over the warp's sub-tile; each warp then walks only the
// entries that touch its sub-tile, with the mask packed into the list word.
// Semantics (renderer.cpp:160-181): per pixel, the contributors are the
// splats whose rect contains it, in (depth, index) order; break before
// compositing once T < stop; alpha = min(o g, clamp); no 1/255 skip. The stop
// decision uses T in FP64 (stacked clamped splats give T = (1 - 0.99)^k
// exactly at the 1e-4 threshold, test_renderer.cpp:272-282).
constexpr int kBlendThreads = 128;
constexpr int kBatch = 256;
constexpr int kBlendWarps = kBlendThreads / 32;

// exp2(-q): the record's factor carries sqrt(log2(e) / 2), so this is
// exp(-q_ref / 2) of renderer.cpp:53-59 (ex2.approx.ftz: ~2 ulp).
__device__ __forceinline__ float ex2_neg(float q) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-q));
    return y;
}

// Hit mask of a splat rect over the 8x8 sub-tile at (sx, sy): low byte = the
// sub-tile columns inside [x0, x1], high byte = the rows inside [y0, y1]; 0
// when they do not overlap. A lane's hit test is then two shifts and an AND.
__device__ __forceinline__ uint32_t span_bits(int lo, int hi) {  // bits [lo, hi] of 0..7, clamped
    lo = max(lo, 0);
    hi = min(hi, 7);
    return lo <= hi ? ((0xffu >> (7 - hi)) & (0xffu << lo)) : 0u;
}

__device__ __forceinline__ uint32_t region_hits(int x0, int x1, int y0, int y1, int sx, int sy) {
    const uint32_t cm = span_bits(x0 - sx, x1 - sx), rm = span_bits(y0 - sy, y1 - sy);
    return cm && rm ? (cm | (rm << 8)) : 0u;
}

// Entry t of a batch into shared memory. The record holds L' = kQScale L
// (minv = L^T L, L upper triangular) and the offsets k' of L'(p - m) written
// around the rect centre o (preprocess.cu); here o moves to the tile origin,
// so t = L'(p - m) at tile-local pixel (lx, ly) is
//   t1 = l11 lx + l12 ly + k1,  t2 = l22 ly + k2
// with every FP32 term of the size of the footprint in pixels (the rect
// centre is within the image, the tile origin within 16 px of the pixel).
// Layout: {l11, l12, l22, k1}, {k2, o, r, g}, {b, target, -, -}.
__device__ __forceinline__ void stage_entry(int t, uint32_t row, const float4* __restrict__ rec, int tx0, int ty0,
                                            float4* s_rec, uint16_t (*s_hm)[kBatch]) {
    const size_t r = 3 * static_cast<size_t>(row);
    const float4 a = rec[r], b = rec[r + 1], c = rec[r + 2];
    int x0, x1, y0, y1;
    unpack_rect(c, x0, x1, y0, y1);
    const float ox = 0.5f * static_cast<float>(x0 + x1) - static_cast<float>(tx0);  // exact
    const float oy = 0.5f * static_cast<float>(y0 + y1) - static_cast<float>(ty0);
    s_rec[3 * t] = make_float4(a.x, a.y, a.z, fmaf(-a.x, ox, fmaf(-a.y, oy, a.w)));
    s_rec[3 * t + 1] = make_float4(fmaf(-a.z, oy, b.x), b.y, b.z, b.w);
    s_rec[3 * t + 2] = make_float4(c.x, c.w, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < kBlendWarps; ++w)
        s_hm[w][t] = static_cast<uint16_t>(region_hits(x0, x1, y0, y1, tx0 + (w & 1) * 8, ty0 + (w >> 1) * 8));
}

// This warp's entries of the batch (hit mask != 0), ascending, as
// (entry | hit mask << 16).
__device__ __forceinline__ int build_list(int warp, int lane, int cnt, const uint16_t (*s_hm)[kBatch],
                                          uint32_t (*s_list)[kBatch]) {
    int nl = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int e = c0 + lane;
        const uint32_t hm = e < cnt ? s_hm[warp][e] : 0u;
        const unsigned bal = __ballot_sync(0xffffffffu, hm != 0);
        if (hm) s_list[warp][nl + __popc(bal & ((1u << lane) - 1u))] = static_cast<uint32_t>(e) | (hm << 16);
        nl += __popc(bal);
    }
    __syncwarp();
    return nl;
}

// One pixel's front-to-back loop over the entries of a 32-entry chunk it
// hits (bit e of m = entry e of the chunk, ascending = compositing order).
struct FwdPix {
    float T, r, g, b;
    double Td;
    uint32_t n, last;
    bool done;
};

__device__ __forceinline__ void fwd_pixel(FwdPix& P, uint32_t m, const uint32_t* __restrict__ list,
                                          const float4* s_rec, float lx, float ly, uint32_t base, double tstop,
                                          float aclamp, double oma_clamp) {
    while (m) {
        const int e = __ffs(m) - 1;
        m &= m - 1;
        if (P.Td < tstop) {
            P.done = true;
            return;
        }
        const uint32_t j = list[e] & 0xffffu;
        BSG_DASSERT(j < kBatch);
        const float4 A = s_rec[3 * j], B = s_rec[3 * j + 1];
        const float cbl = s_rec[3 * j + 2].x;
        const float t1 = fmaf(A.y, ly, fmaf(A.x, lx, A.w)), t2 = fmaf(A.z, ly, B.x);
        const float og = B.y * ex2_neg(fmaf(t1, t1, t2 * t2));
        const bool clamped = og >= aclamp;  // no float lies in [0.99, float(0.99))
        const float alpha = clamped ? aclamp : og;
        const float w = alpha * P.T;
        P.r = fmaf(B.z, w, P.r);
        P.g = fmaf(B.w, w, P.g);
        P.b = fmaf(cbl, w, P.b);
        P.T *= 1.f - alpha;
        P.Td *= clamped ? oma_clamp : static_cast<double>(1.f - og);  // 1 - og exact for og >= 0.5
        ++P.n;
        P.last = base + j;
    }
}

// The forward walks each pixel's own contributors: per 32-entry chunk of the
// warp's list, 16 ballots give every lane the chunk's column and row masks
// over its sub-tile, their AND is the set of entries whose rect contains the
// lane's pixel, and the lane loops over those set bits. Lanes of a warp are
// busy whenever their pixel has a contributor left in the chunk (a per-entry
// warp loop idles every lane outside the entry's rect).
__global__ __launch_bounds__(kBlendThreads, 8) void blend_fwd_kernel(const uint2* __restrict__ ranges,
                                                                  const uint32_t* __restrict__ pval,
                                                                  const float4* __restrict__ rec, int W, int H,
                                                                  int tiles_x, double tstop, float aclamp,
                                                                  double aclamp_d, float bg0, float bg1, float bg2,
                                                                  float* __restrict__ out_rgb,
                                                                  float* __restrict__ out_T,
                                                                  uint32_t* __restrict__ out_n,
                                                                  uint32_t* __restrict__ out_last,
                                                                  unsigned long long* __restrict__ evals,
                                                                  const uint32_t* __restrict__ tile_order) {
    pdl_prologue();
    __shared__ float4 s_rec[3 * kBatch];
    __shared__ uint16_t s_hm[kBlendWarps][kBatch];
    __shared__ uint32_t s_list[kBlendWarps][kBatch];
    const int tile = static_cast<int>(tile_order[blockIdx.x]);
    const int tx0 = (tile % tiles_x) * kTile, ty0 = (tile / tiles_x) * kTile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lxi = (warp & 1) * 8 + (lane & 7), ly0i = (warp >> 1) * 8 + (lane >> 3);
    const int px = tx0 + lxi, py0 = ty0 + ly0i, py1 = py0 + 4;
    const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
    const float lx = static_cast<float>(lxi), ly0 = static_cast<float>(ly0i), ly1 = ly0 + 4.f;
    const int hc = lane & 7, hr = lane >> 3;  // this lane's sub-tile column, first row
    const uint2 range = ranges[tile];
    BSG_DASSERT(range.x <= range.y);
    const double oma_clamp = 1.0 - aclamp_d;
    FwdPix P0{1.f, 0.f, 0.f, 0.f, 1.0, 0u, 0u, !in0}, P1{1.f, 0.f, 0.f, 0.f, 1.0, 0u, 0u, !in1};
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        if (__syncthreads_count(P0.done && P1.done) == kBlendThreads) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t idx = start + threadIdx.x + h * kBlendThreads;
            if (idx < range.y) stage_entry(threadIdx.x + h * kBlendThreads, pval[idx], rec, tx0, ty0, s_rec, s_hm);
        }
        __syncthreads();
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kBatch), range.y - start));
        // a warp whose pixels have all stopped skips the batch (the CTA leaves
        // once every warp has)
        const int nl = __all_sync(0xffffffffu, P0.done && P1.done) ? 0 : build_list(warp, lane, cnt, s_hm, s_list);
        const uint32_t base = start - range.x + 1;  // 1-based list position of entry 0 of the batch
        for (int c0 = 0; c0 < nl; c0 += 32) {
            const uint32_t hm = c0 + lane < nl ? s_list[warp][c0 + lane] >> 16 : 0u;
            uint32_t mc = 0, mr0 = 0, mr1 = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t b = __ballot_sync(0xffffffffu, (hm >> c) & 1u);
                mc = c == hc ? b : mc;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t b = __ballot_sync(0xffffffffu, (hm >> (8 + r)) & 1u);
                mr0 = r == hr ? b : mr0;
                mr1 = r == hr + 4 ? b : mr1;
            }
            const uint32_t* list = &s_list[warp][c0];
            if (!P0.done) fwd_pixel(P0, mc & mr0, list, s_rec, lx, ly0, base, tstop, aclamp, oma_clamp);
            if (!P1.done) fwd_pixel(P1, mc & mr1, list, s_rec, lx, ly1, base, tstop, aclamp, oma_clamp);
        }
        __syncwarp();
    }
    // work counter for the FP32 roofline: composited (pixel, contributor) pairs
    uint32_t ev = P0.n + P1.n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
    if (lane == 0 && ev) atomicAdd(evals, static_cast<unsigned long long>(ev));
    if (in0) {
        const size_t p = static_cast<size_t>(py0) * W + px;
        out_rgb[3 * p + 0] = P0.r + P0.T * bg0;
        out_rgb[3 * p + 1] = P0.g + P0.T * bg1;
        out_rgb[3 * p + 2] = P0.b + P0.T * bg2;
        out_T[p] = static_cast<float>(P0.Td);
        out_n[p] = P0.n;
        out_last[p] = P0.last;
    }
    if (in1) {
        const size_t p = static_cast<size_t>(py1) * W + px;
        out_rgb[3 * p + 0] = P1.r + P1.T * bg0;
        out_rgb[3 * p + 1] = P1.g + P1.T * bg1;
        out_rgb[3 * p + 2] = P1.b + P1.T * bg2;
        out_T[p] = static_cast<float>(P1.Td);
        out_n[p] = P1.n;
        out_last[p] = P1.last;
    }
}

// Warp sum of 9 per-lane values as a transposition: at each xor stage a
// lane keeps one half of its (zero-padded) array and adds the partner's copy
// of the same half, so 5 + 3 + 2 + 1 + 1 = 12 shuffles give every lane the
// full sum of value index reduced9_index(lane) (valid when < 9; lanes that
// differ only in bit 0 hold the same value).
__device__ __forceinline__ float pair_stage(float keep_lo, float keep_hi, bool hi, int mask) {
    const float send = hi ? keep_lo : keep_hi;
    const float keep = hi ? keep_hi : keep_lo;
    return keep + __shfl_xor_sync(0xffffffffu, send, mask);
}

__device__ __forceinline__ float warp_reduce9(const float (&v)[9], int lane) {
    const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
    float a1[5];
#pragma unroll
    for (int j = 0; j < 4; ++j) a1[j] = pair_stage(v[2 * j], v[2 * j + 1], b16, 16);
    a1[4] = pair_stage(v[8], 0.f, b16, 16);
    float a2[3];
#pragma unroll
    for (int j = 0; j < 2; ++j) a2[j] = pair_stage(a1[2 * j], a1[2 * j + 1], b8, 8);
    a2[2] = pair_stage(a1[4], 0.f, b8, 8);
    const float a30 = pair_stage(a2[0], a2[1], b4, 4);
    const float a31 = pair_stage(a2[2], 0.f, b4, 4);
    const float a4 = pair_stage(a30, a31, b2, 2);
    return a4 + __shfl_xor_sync(0xffffffffu, a4, 1);
}

// Value index owned by `lane` after warp_reduce9.
__device__ __forceinline__ int reduced9_index(int lane) {
    return ((lane & 2) ? 8 : 0) + ((lane & 4) ? 4 : 0) + ((lane & 8) ? 2 : 0) + ((lane & 16) ? 1 : 0);
}

// Per-pixel reverse recurrence (renderer.cpp:288-308) for one contributor.
// The colour suffix enters dL/dalpha only through its dot product with the
// pixel's dL/dC, so that dot product (ds) is carried instead of the 3-vector:
//   dL/dalpha = dL/dC . (c T_before - s / (1 - alpha))
//             = T_before (dL/dC . c) - ds / (1 - alpha),   ds += (dL/dC . c) alpha T_before.
struct BwdPix {
    float T, d0, d1, d2, ds;
};

// Accumulators: 0,1 k L'^T L'd (mean); 2,3,4 k (L'^T L'd)(L'^T L'd)^T (cov, no
// 1/2); 5,6,7 colour; 8 opacity -- rescaled by the fold (unscale_g2d).
__device__ __forceinline__ void bwd_step(BwdPix& P, float u, float ly, const float4& A, const float4& B, float cbl,
                                         float aclamp, float (&acc)[9]) {
    const float t1 = fmaf(A.y, ly, u), t2 = fmaf(A.z, ly, B.x);
    const float g = ex2_neg(fmaf(t1, t1, t2 * t2));
    const float og = B.y * g;
    const float alpha = fminf(og, aclamp);
    const float inv = fast_rcp(1.f - alpha);  // 1 - alpha >= 0.01
    const float Tb = P.T * inv;
    const float at = alpha * Tb;
    acc[5] = fmaf(P.d0, at, acc[5]);
    acc[6] = fmaf(P.d1, at, acc[6]);
    acc[7] = fmaf(P.d2, at, acc[7]);
    const float dc = fmaf(P.d0, B.z, fmaf(P.d1, B.w, P.d2 * cbl));
    const float dlda = fmaf(Tb, dc, -(inv * P.ds));
    if (og < aclamp) {
        const float kk = dlda * og;
        const float mdx = A.x * t1, mdy = fmaf(A.y, t1, A.z * t2);  // L'^T t
        const float u0 = kk * mdx, u1 = kk * mdy;
        acc[0] += u0;
        acc[1] += u1;
        acc[2] = fmaf(u0, mdx, acc[2]);
        acc[3] = fmaf(u0, mdy, acc[3]);
        acc[4] = fmaf(u1, mdy, acc[4]);
        acc[8] = fmaf(dlda, g, acc[8]);
    }
    P.ds = fmaf(dc, at, P.ds);
    P.T = Tb;
}

// K9 blend backward: reverse traversal of each pixel's composited list
// (T recovered by division, 1 - alpha >= 0.01), same CTA layout, staging and
// per-warp lists as K7. The 9 per-splat gradients of the warp's 64 pixels are
// summed in registers, transpose-reduced across the warp in 12 shuffles and
// added with 9 scalar atomics; up to kDirectLanes contributing lanes add
// their own values directly with vector atomics instead (no shuffles). The
// threshold trades issue slots against L2 atomic traffic: measured at cfg 2,
// blend bwd 0.178 / 0.173 / 0.165 / 0.156 / 0.158 / 0.186 / 0.295 ms for
// 2 / 4 / 8 / 16 / 20 / 24 / 32 lanes; one butterfly stage with the lower 16
// lanes adding directly (fewer shuffles, more atomics) was slower still.
constexpr int kDirectLanes = 16;

__global__ __launch_bounds__(kBlendThreads, 8) void blend_bwd_kernel(const uint2* __restrict__ ranges,
                                                                  const uint32_t* __restrict__ pval,
                                                                  const float4* __restrict__ rec, int W, int H,
                                                                  int tiles_x, float aclamp, float bg0, float bg1,
                                                                  float bg2, const float* __restrict__ in_T,
                                                                  const uint32_t* __restrict__ in_last,
                                                                  const float* __restrict__ dl_dc,
                                                                  float4* __restrict__ g2d,
                                                                  double* __restrict__ g2d_wide,
                                                                  const uint32_t* __restrict__ tile_order,
                                                                  int direct_lanes) {
    pdl_prologue();
    __shared__ float4 s_rec[3 * kBatch];
    __shared__ uint16_t s_hm[kBlendWarps][kBatch];
    __shared__ uint32_t s_list[kBlendWarps][kBatch];
    __shared__ uint32_t s_max;
    const int tile = static_cast<int>(tile_order[blockIdx.x]);
    const int tx0 = (tile % tiles_x) * kTile, ty0 = (tile / tiles_x) * kTile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lxi = (warp & 1) * 8 + (lane & 7), ly0i = (warp >> 1) * 8 + (lane >> 3);
    const int px = tx0 + lxi, py0 = ty0 + ly0i, py1 = py0 + 4;
    const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
    const float lx = static_cast<float>(lxi), ly0 = static_cast<float>(ly0i), ly1 = ly0 + 4.f;
    // this lane's two pixels in a hit mask: column bit | row bit
    const uint32_t hit_bits0 = (1u << (lane & 7)) | (1u << (8 + (lane >> 3)));
    const uint32_t hit_bits1 = (1u << (lane & 7)) | (1u << (12 + (lane >> 3)));
    const uint2 range = ranges[tile];
    BwdPix P0{1.f, 0.f, 0.f, 0.f, 0.f}, P1{1.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t last0 = 0, last1 = 0;
    if (in0) {
        const size_t p = static_cast<size_t>(py0) * W + px;
        last0 = in_last[p];
        P0.T = in_T[p];
        P0.d0 = dl_dc[3 * p]; P0.d1 = dl_dc[3 * p + 1]; P0.d2 = dl_dc[3 * p + 2];
    }
    if (in1) {
        const size_t p = static_cast<size_t>(py1) * W + px;
        last1 = in_last[p];
        P1.T = in_T[p];
        P1.d0 = dl_dc[3 * p]; P1.d1 = dl_dc[3 * p + 1]; P1.d2 = dl_dc[3 * p + 2];
    }
    // suffix behind the last contributor: T_final bg (renderer.cpp:282-286)
    P0.ds = P0.T * fmaf(P0.d0, bg0, fmaf(P0.d1, bg1, P0.d2 * bg2));
    P1.ds = P1.T * fmaf(P1.d0, bg0, fmaf(P1.d1, bg1, P1.d2 * bg2));
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    uint32_t wm = max(last0, last1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (lane == 0) atomicMax(&s_max, wm);
    __syncthreads();
    const uint32_t max_last = s_max;
    for (int end = static_cast<int>(max_last); end > 0; end -= kBatch) {
        const int start = end - kBatch > 0 ? end - kBatch : 0;
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = threadIdx.x + h * kBlendThreads;
            if (start + t < end) stage_entry(t, pval[range.x + start + t], rec, tx0, ty0, s_rec, s_hm);
        }
        __syncthreads();
        // entries at or past this warp's largest `last` touch none of its pixels
        const int nl = build_list(warp, lane, max(0, min(end, static_cast<int>(wm)) - start), s_hm, s_list);
        for (int k = nl - 1; k >= 0; --k) {
            const uint32_t wd = s_list[warp][k];
            const uint32_t sj = wd & 0xffffu, hm = wd >> 16;
            const uint32_t j = static_cast<uint32_t>(start) + sj;  // 0-based list position
            const bool hit0 = j < last0 && (hm & hit_bits0) == hit_bits0;
            const bool hit1 = j < last1 && (hm & hit_bits1) == hit_bits1;
            const unsigned mask = __ballot_sync(0xffffffffu, hit0 || hit1);
            if (mask == 0) continue;
            const float4 A = s_rec[3 * sj], B = s_rec[3 * sj + 1];
            const float2 C = *reinterpret_cast<const float2*>(&s_rec[3 * sj + 2]);
            const float u = fmaf(A.x, lx, A.w);
            float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (hit0) bwd_step(P0, u, ly0, A, B, C.x, aclamp, acc);
            if (hit1) bwd_step(P1, u, ly1, A, B, C.x, aclamp, acc);
            const uint32_t target = __float_as_uint(C.y);  // row, or kWideBit | FP64 slot (kWideArea)
            const bool wide = target & kWideBit;
            BSG_DASSERT(sj < kBatch && (wide ? (target & ~kWideBit) < kWideCap : true));
            float* dst = reinterpret_cast<float*>(g2d + 3 * static_cast<size_t>(target & ~kWideBit));
            if (__popc(mask) <= direct_lanes && !wide) {
                if (hit0 || hit1) {
                    atomicAdd(reinterpret_cast<float4*>(dst), make_float4(acc[0], acc[1], acc[2], acc[3]));
                    atomicAdd(reinterpret_cast<float4*>(dst) + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
                    atomicAdd(dst + 8, acc[8]);
                }
            } else {
                const float r = warp_reduce9(acc, lane);
                if (!wide) {
                    // values 0-3 / 4-7 sit in lanes {0,16,8,24} / {4,20,12,28}, value 8
                    // in lane 2: three shuffles gather the quads into lanes 0 and 4,
                    // so the sum reaches L2 as 3 vector atomics instead of 9 scalar
                    const float q1 = __shfl_down_sync(0xffffffffu, r, 16);
                    const float q2 = __shfl_down_sync(0xffffffffu, r, 8);
                    const float q3 = __shfl_down_sync(0xffffffffu, r, 24);
                    if ((lane & ~4) == 0) atomicAdd(reinterpret_cast<float4*>(dst + lane), make_float4(r, q1, q2, q3));
                    if (lane == 2) atomicAdd(dst + 8, r);
                } else {
                    const int idx = reduced9_index(lane);
                    if ((lane & 1) == 0 && idx < 9)
                        atomicAdd(g2d_wide + 9 * static_cast<size_t>(target & ~kWideBit) + idx, static_cast<double>(r));
                }
            }
        }
    }
}

}  // namespace

void launch_pairs(Ctx* c, const DevCam& cam, uint32_t V) {
    if (V == 0) return;
    const uint32_t ntiles = static_cast<uint32_t>(cam.tiles_x * cam.tiles_y);
    launch_pdl(c->stream, (V + 255) / 256, 256, 0, emit_pairs_kernel, c->vrow[c->depth_sorted], c->poff, c->rec, V, cam.tiles_x,
                                                              c->pkey[0], c->pval[0], static_cast<uint32_t>(c->pcap),
                                                              &c->counters->tile_hist[0][0], c->ranges, ntiles);
    BSG_LAUNCHED(c);
}

// V > 0: the pair emission already cleared the tile ranges.
void launch_ranges(Ctx* c, const DevCam& cam, uint32_t V, uint32_t P) {
    const size_t ntiles = static_cast<size_t>(cam.tiles_x) * cam.tiles_y;
    if (V == 0) BSG_CUDA(cudaMemsetAsync(c->ranges, 0, ntiles * sizeof(uint2), c->stream));
    if (P == 0) {
        launch_pdl(c->stream, 1, 1024, 0, tile_order_kernel, c->ranges, static_cast<uint32_t>(ntiles), c->tile_order);
        BSG_LAUNCHED(c);
        return;
    }
    launch_pdl(c->stream, (P + 255) / 256, 256, 0, ranges_kernel, c->pkey[c->pairs_sorted], P, c->ranges);
    BSG_LAUNCHED(c);
    launch_pdl(c->stream, 1, 1024, 0, tile_order_kernel, c->ranges, static_cast<uint32_t>(ntiles), c->tile_order);
    BSG_LAUNCHED(c);
}

void launch_tile_scan(Ctx* c, const DevCam& cam, uint32_t seq) {
    const uint32_t ntiles = static_cast<uint32_t>(cam.tiles_x * cam.tiles_y);
    if (ntiles > 1024u) {  // several CTAs (scan.cu)
        launch_tile_scan_multi(c, ntiles, seq);
        return;
    }
    launch_pdl(c->stream, 1, 1024, 0, tile_scan_kernel, c->tile_cnt, ntiles, c->ranges, c->tile_cur, c->tile_order,
               c->mbox, seq, &c->counters->pairs);
    BSG_LAUNCHED(c);
}

void launch_emit_tiles(Ctx* c, const DevCam& cam) {
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(static_cast<uint32_t>((c->n + 255) / 256), 148 * 8));
    launch_pdl(c->stream, grid, 256, 0, emit_tiles_kernel, c->vis_rows, c->counters, c->rec, cam.tiles_x, c->tile_cur,
               c->pval[1], static_cast<uint32_t>(c->pcap), c->ranges);
    BSG_LAUNCHED(c);
}

void launch_tile_sort(Ctx* c, const DevCam& cam, uint32_t max_tile) {
    const uint32_t ntiles = static_cast<uint32_t>(cam.tiles_x * cam.tiles_y);
    uint32_t N = 2;
    while (N < max_tile) N <<= 1;
    const size_t smem = N * (sizeof(uint64_t) + sizeof(uint32_t));  // packed keys (+ rows for the full-key re-sort)
    static bool attr_set[64] = {};
    if (!attr_set[c->device]) {
        BSG_CUDA(cudaFuncSetAttribute(tile_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kTileSortCap * (sizeof(uint64_t) + sizeof(uint32_t)))));
        attr_set[c->device] = true;
    }
    // 128 threads: one compare-exchange per thread per stage for tiles up to
    // 256 pairs (the common case), a few for the long ones, launched first
    launch_pdl(c->stream, ntiles, kTileSortThreads, smem, tile_sort_kernel, c->ranges, c->tile_order, c->pval[1], c->depth_key,
               c->pval[0]);
    BSG_LAUNCHED(c);
}

void launch_blend_fwd(Ctx* c, const DevCam& cam, const DevRender& rc) {
    const int ntiles = cam.tiles_x * cam.tiles_y;
    launch_pdl(c->stream, ntiles, kBlendThreads, 0, blend_fwd_kernel, c->ranges, c->pval[c->pairs_sorted], c->rec, cam.W, cam.H, cam.tiles_x, rc.tstop,
        static_cast<float>(rc.alpha_clamp), rc.alpha_clamp, rc.bg[0], rc.bg[1], rc.bg[2], c->out_rgb, c->out_T,
        c->out_n, c->out_last, &c->counters->evals, c->tile_order);
    BSG_LAUNCHED(c);
}

// BSG_DIRECT_LANES overrides kDirectLanes (measurement only)
static int direct_lanes() {
    static const int v = [] {
        const char* e = std::getenv("BSG_DIRECT_LANES");
        return e ? std::atoi(e) : kDirectLanes;
    }();
    return v;
}

void launch_blend_bwd(Ctx* c, const DevCam& cam, const DevRender& rc) {
    const int ntiles = cam.tiles_x * cam.tiles_y;
    launch_pdl(c->stream, ntiles, kBlendThreads, 0, blend_bwd_kernel, c->ranges, c->pval[c->pairs_sorted], c->rec, cam.W, cam.H, cam.tiles_x, static_cast<float>(rc.alpha_clamp),
        rc.bg[0], rc.bg[1], rc.bg[2], c->out_T, c->out_last, c->dl_dc, c->g2d, c->g2d_wide, c->tile_order,
        direct_lanes());
    BSG_LAUNCHED(c);
}

}  // namespace bsg
