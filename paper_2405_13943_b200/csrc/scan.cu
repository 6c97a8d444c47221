// Single-pass exclusive scan with decoupled look-back, and the stable
// compaction of visible splats built on it. Both are HBM-bound streaming
// passes: one read of the input, one write of the output.
#include <cstddef>

#include "bsg_internal.cuh"

#include <atomic>

namespace bsg {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr uint32_t kFlagAgg = 1u, kFlagInc = 2u;

// Status word: [epoch 30 | flag 2 | value 32]. A word from another launch
// (other epoch) reads as "not yet published", so the buffer is never cleared.
__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, uint32_t flag, uint32_t v) {
    return (static_cast<unsigned long long>(epoch) << 34) | (static_cast<unsigned long long>(flag) << 32) | v;
}

__device__ __forceinline__ void publish(unsigned long long* st, uint32_t epoch, uint32_t flag, uint32_t v) {
    atomicExch(st, pack_status(epoch, flag, v));
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
        if (lane == kScanThreads / 32 - 1) *total = wi;
    }
    __syncthreads();
    return s_warp[warp] + inc - v;
}

// block_exclusive for a 1024-thread block (32 warps).
__device__ __forceinline__ uint32_t block_exclusive_1024(uint32_t v, uint32_t* s_warp, uint32_t* total) {
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
        s_warp[lane] = wi - w;
        if (lane == 31) *total = wi;
    }
    __syncthreads();
    return s_warp[warp] + inc - v;
}

// Warp 0 walks predecessors 32 at a time until it meets an inclusive prefix.
__device__ __forceinline__ uint32_t look_back(unsigned long long* status, uint32_t tile, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    uint32_t prefix = 0;
    int64_t window = static_cast<int64_t>(tile) - 1;
    while (window >= 0) {
        const int64_t p = window - lane;
        unsigned long long st = 0;
        uint32_t flag = kFlagInc;  // lanes past tile 0 act as an empty inclusive prefix
        if (p >= 0) {
            do {
                st = *reinterpret_cast<volatile unsigned long long*>(&status[p]);
                flag = static_cast<uint32_t>(st >> 34) == epoch ? static_cast<uint32_t>(st >> 32) & 3u : 0u;
            } while (flag == 0);
        }
        const uint32_t inc_mask = __ballot_sync(0xffffffffu, flag == kFlagInc);
        const int stop = __ffs(inc_mask) - 1;  // nearest predecessor with an inclusive prefix
        uint32_t val = (p >= 0 && (inc_mask == 0 || lane <= stop)) ? static_cast<uint32_t>(st) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (inc_mask != 0) break;
        window -= 32;
    }
    return prefix;
}

// MODE 0: plain exclusive scan of in[gather ? gather[i] : i].
// MODE 1: compaction of rows with tiles[i] > 0 (in = tiles), emits the FP64
//         depth bits as u64 keys + rows, 8 digit histograms.
// MODE 2: as 1 with the 32-bit range-normalised key (bits - zmin) >> shift
//         (depth_key_bits(V) <= 32 bits), no histograms.
template <int MODE>
__global__ __launch_bounds__(kScanThreads) void scan_kernel(const uint32_t* __restrict__ in,
                                                            const uint32_t* __restrict__ gather,
                                                            uint32_t* __restrict__ out, uint32_t n,
                                                            unsigned long long* status, Lookback lb, Publish pub,
                                                            uint32_t* total_out, const uint64_t* __restrict__ keys,
                                                            void* __restrict__ out_keys_v,
                                                            const StepCounters* __restrict__ range,
                                                            uint32_t* __restrict__ out_rows,
                                                            uint32_t* __restrict__ hist_out, int hist_first,
                                                            uint32_t* __restrict__ mask_out, uint32_t mask_words,
                                                            uint32_t* __restrict__ prefix_out) {
    pdl_prologue();
    __shared__ uint32_t s_tile, s_prefix, s_total;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    constexpr int kDigits = 8;
    __shared__ uint32_t s_hist[MODE == 1 ? kDigits * 256 : 1];
    if (threadIdx.x == 0) s_tile = static_cast<uint32_t>(atomicAdd(lb.ticket, 1ull) - lb.base);
    if (MODE == 1)
        for (int k = threadIdx.x; k < kDigits * 256; k += kScanThreads) s_hist[k] = 0;
    unsigned long long zmin = 0;
    int shift = 0;
    if (MODE == 2) {
        zmin = ~range->zmin_inv;
        const unsigned long long span = range->zmax - zmin;  // 0 when nothing (or one depth) is visible
        const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
        const int kb = depth_key_bits(range->visible_pre);
        shift = bits > kb ? bits - kb : 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = static_cast<uint64_t>(tile) * kScanTile + static_cast<uint64_t>(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        uint32_t x = 0;
        if (i < n) {
            if (MODE != 0) {
                x = in[i] > 0 ? 1u : 0u;
            } else {
                x = in[gather ? gather[i] : i];
            }
        }
        v[k] = x;
        sum += x;
    }
    if (MODE != 0) {
        // 1 bit per row: this thread's kScanItems rows are kScanItems bits of a
        // 32-row word, kLanesPerWord consecutive lanes fill one word
        static_assert(32 % kScanItems == 0, "rows per thread must divide a mask word");
        constexpr int kLanesPerWord = 32 / kScanItems;
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) bits |= v[k] << k;
        uint32_t wbits = bits;
#pragma unroll
        for (int l = 1; l < kLanesPerWord; ++l) wbits |= __shfl_down_sync(0xffffffffu, bits, l) << (kScanItems * l);
        const uint64_t word = base / 32;
        if ((threadIdx.x % kLanesPerWord) == 0 && word < mask_words) mask_out[word] = wbits;
    }
    const uint32_t tprefix = block_exclusive(sum, s_warp, &s_total);
    if (threadIdx.x < 32) {
        const uint32_t total = s_total;
        if (tile == 0) {
            if (threadIdx.x == 0) {
                publish(&status[0], lb.epoch, kFlagInc, total);
                s_prefix = 0;
            }
        } else {
            if (threadIdx.x == 0) publish(&status[tile], lb.epoch, kFlagAgg, total);
            const uint32_t prefix = look_back(status, tile, lb.epoch);
            if (threadIdx.x == 0) {
                publish(&status[tile], lb.epoch, kFlagInc, prefix + total);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && (static_cast<uint64_t>(tile) + 1) * kScanTile >= n) {
        const uint32_t grand = s_prefix + s_total;
        if (total_out) *total_out = grand;
        if (pub.seq_word) {  // host-mapped mailbox: value(s), system fence, sequence word
            *reinterpret_cast<volatile uint32_t*>(pub.val) = grand;
            if (pub.extra_dst) *reinterpret_cast<volatile uint32_t*>(pub.extra_dst) = *pub.extra_src;
            __threadfence_system();
            *reinterpret_cast<volatile uint32_t*>(pub.seq_word) = pub.seq;
        }
    }
    uint32_t run = s_prefix + tprefix;
    const int lane = threadIdx.x & 31;
    if (MODE != 0 && (threadIdx.x % (32 / kScanItems)) == 0 && base / 32 < mask_words)
        prefix_out[base / 32] = run;  // visible rows before this 32-row word
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        if (MODE != 0) {
            const bool vis = v[k] != 0;  // v[k] = 0 past n
            uint64_t key = 0;
            if (vis) {
                const uint64_t zb = keys[i];
                if (MODE == 2) {
                    key = (zb - zmin) >> shift;
                    static_cast<uint32_t*>(out_keys_v)[run] = static_cast<uint32_t>(key);
                } else {
                    key = zb;
                    static_cast<uint64_t*>(out_keys_v)[run] = key;
                }
                out_rows[run] = static_cast<uint32_t>(i);
                out[run] = static_cast<uint32_t>(i);
            }
            // digit histograms (the FP64-bits fall-back only; the 32-bit keys get
            // theirs from a pass over the V compacted keys, radix.cu): the upper
            // digits are nearly constant, so lanes whose digit equals the first
            // active lane's are counted with one atomic (ballot), the rest add
            // individually
            const unsigned act = MODE == 1 ? __ballot_sync(0xffffffffu, vis) : 0u;
            if (act) {
                const int src = __ffs(act) - 1;
#pragma unroll
                for (int p = 0; p < kDigits; ++p) {
                    if (p < hist_first) continue;
                    const uint32_t d = static_cast<uint32_t>((key >> (8 * p)) & 0xffu);
                    const uint32_t d0 = __shfl_sync(0xffffffffu, d, src);
                    const unsigned same = __ballot_sync(0xffffffffu, vis && d == d0);
                    if (lane == src) atomicAdd(&s_hist[p * 256 + d0], __popc(same));
                    else if (vis && d != d0) atomicAdd(&s_hist[p * 256 + d], 1u);
                }
            }
        } else if (i < n) {
            out[i] = run;
        }
        run += v[k];
    }
    if (MODE == 1) {
        __syncthreads();
        for (int k = threadIdx.x; k < kDigits * 256; k += kScanThreads)
            if (s_hist[k]) atomicAdd(&hist_out[k], s_hist[k]);
    }
}

// Compaction of the visible rows from the 1-bit-per-row visibility mask the
// preprocess writes (per-tile binning path: no depth keys needed): 2 mask
// words (64 rows) per thread, decoupled look-back across CTAs, each thread's
// visible rows written in ascending order. Reads n / 8 bytes instead of the
// 4-byte tile count of every row. (cfg 3: 8 / 4 / 2 words per thread -> 92 /
// 184 / 367 CTAs, 16.6 / 16.0 / 15.8 us.)
constexpr int kMaskItems = 2;
constexpr int kMaskTile = kScanThreads * kMaskItems;  // words per CTA
__global__ __launch_bounds__(kScanThreads) void compact_mask_kernel(const uint32_t* __restrict__ mask, uint32_t nwords,
                                                                    unsigned long long* status, Lookback lb,
                                                                    Publish pub, uint32_t* total_out,
                                                                    uint32_t* __restrict__ out_rows) {
    pdl_prologue();
    __shared__ uint32_t s_tile, s_prefix, s_total;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    if (threadIdx.x == 0) s_tile = static_cast<uint32_t>(atomicAdd(lb.ticket, 1ull) - lb.base);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t w0 = static_cast<uint64_t>(tile) * kMaskTile + static_cast<uint64_t>(threadIdx.x) * kMaskItems;
    uint32_t wv[kMaskItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kMaskItems; ++k) {
        wv[k] = w0 + k < nwords ? mask[w0 + k] : 0u;
        sum += __popc(wv[k]);
    }
    const uint32_t tprefix = block_exclusive(sum, s_warp, &s_total);
    if (threadIdx.x < 32) {
        const uint32_t total = s_total;
        if (tile == 0) {
            if (threadIdx.x == 0) {
                publish(&status[0], lb.epoch, kFlagInc, total);
                s_prefix = 0;
            }
        } else {
            if (threadIdx.x == 0) publish(&status[tile], lb.epoch, kFlagAgg, total);
            const uint32_t prefix = look_back(status, tile, lb.epoch);
            if (threadIdx.x == 0) {
                publish(&status[tile], lb.epoch, kFlagInc, prefix + total);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && (static_cast<uint64_t>(tile) + 1) * kMaskTile >= nwords) {
        const uint32_t grand = s_prefix + s_total;
        if (total_out) *total_out = grand;
        if (pub.seq_word) {  // host-mapped mailbox: value(s), system fence, sequence word
            *reinterpret_cast<volatile uint32_t*>(pub.val) = grand;
            if (pub.extra_dst) *reinterpret_cast<volatile uint32_t*>(pub.extra_dst) = *pub.extra_src;
            __threadfence_system();
            *reinterpret_cast<volatile uint32_t*>(pub.seq_word) = pub.seq;
        }
    }
    uint32_t run = s_prefix + tprefix;
#pragma unroll
    for (int k = 0; k < kMaskItems; ++k) {
        uint32_t b = wv[k];
        const uint32_t row0 = static_cast<uint32_t>((w0 + k) * 32);
        while (b) {
            out_rows[run++] = row0 + (__ffs(b) - 1);
            b &= b - 1;
        }
    }
}

// Per-tile binning, multi-CTA: 1024 tiles per CTA. Pass A: each tile's pair
// range and its kTileSub sub-cursors from an exclusive scan of the tile
// counts (decoupled look-back across CTAs); the launch-order histogram, the
// largest tile and the total; the last CTA publishes P, the largest tile and
// the capacity flag to the mailbox (every predecessor's contributions are in
// by then: each adds them before publishing its aggregate). Pass B: the
// launch order (tiles by descending count, order inside a bucket free), each
// CTA placing its tiles through per-bucket ranges reserved with one atomic
// per bucket.
constexpr int kTileScanThreads = 1024;
__global__ __launch_bounds__(kTileScanThreads) void tile_scan_a_kernel(const uint32_t* __restrict__ cnt, uint32_t ntiles,
                                                                      uint2* __restrict__ ranges,
                                                                      uint32_t* __restrict__ cur,
                                                                      unsigned long long* status, Lookback lb,
                                                                      StepCounters* __restrict__ counters, Mailbox* mb,
                                                                      uint32_t seq) {
    pdl_prologue();
    __shared__ uint32_t s_tile, s_prefix, s_total, s_max;
    __shared__ uint32_t s_warp[kTileScanThreads / 32];
    __shared__ uint32_t s_hist[1024];
    __shared__ unsigned long long s_wide;
    const uint32_t t = threadIdx.x;
    s_hist[t] = 0;
    if (t == 0) {
        s_tile = static_cast<uint32_t>(atomicAdd(lb.ticket, 1ull) - lb.base);
        s_max = 0;
        s_wide = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile, i = tile * kTileScanThreads + t;
    static_assert(kTileSub == 4, "one uint4 of sub-counts per tile");
    const uint4 sc = i < ntiles ? reinterpret_cast<const uint4*>(cnt)[i] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t v = sc.x + sc.y + sc.z + sc.w;
    if (i < ntiles) atomicAdd(&s_hist[1023u - min(v, 1023u)], 1u);
    uint32_t mx = v;
    unsigned long long wide = v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        wide += __shfl_xor_sync(0xffffffffu, wide, o);
    }
    if ((t & 31) == 0) {
        atomicMax(&s_max, mx);
        atomicAdd(&s_wide, wide);
    }
    const uint32_t ex = block_exclusive_1024(v, s_warp, &s_total);  // (its barriers order the shared atomics above)
    // this CTA's contributions to the bucket counts, the largest tile and the
    // wide total, before its aggregate is published
    if (s_hist[t]) atomicAdd(&counters->order_hist[t], s_hist[t]);
    if (t == 0) {
        atomicMax(&counters->tile_max, s_max);
        atomicAdd(&counters->pairs_wide, s_wide);
    }
    __threadfence();
    __syncthreads();
    if (t < 32) {
        const uint32_t total = s_total;
        if (tile == 0) {
            if (t == 0) {
                publish(&status[0], lb.epoch, kFlagInc, total);
                s_prefix = 0;
            }
        } else {
            if (t == 0) publish(&status[tile], lb.epoch, kFlagAgg, total);
            const uint32_t prefix = look_back(status, tile, lb.epoch);
            if (t == 0) {
                publish(&status[tile], lb.epoch, kFlagInc, prefix + total);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    if (i < ntiles) {
        const uint32_t b = s_prefix + ex;
        ranges[i] = make_uint2(b, b + v);
        reinterpret_cast<uint4*>(cur)[i] = make_uint4(b, b + sc.x, b + sc.x + sc.y, b + sc.x + sc.y + sc.z);
    }
    if (t == 0 && (static_cast<uint64_t>(tile) + 1) * kTileScanThreads >= ntiles) {
        // the last CTA: all predecessors' aggregates (and so their atomics) are in
        __threadfence();
        const uint32_t P = s_prefix + s_total;
        counters->pairs = P;
        const uint32_t tmax = *reinterpret_cast<volatile uint32_t*>(&counters->tile_max);
        const unsigned long long pw = *reinterpret_cast<volatile unsigned long long*>(&counters->pairs_wide);
        *reinterpret_cast<volatile uint32_t*>(&mb->P) = P;
        *reinterpret_cast<volatile uint32_t*>(&mb->max_tile) = tmax;
        *reinterpret_cast<volatile uint32_t*>(&mb->pairs_big) = pw >= kMaxPairs ? 1u : 0u;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&mb->seq_p) = seq;
    }
}

__global__ __launch_bounds__(kTileScanThreads) void tile_scan_b_kernel(const uint32_t* __restrict__ cnt, uint32_t ntiles,
                                                                      StepCounters* __restrict__ counters,
                                                                      uint32_t* __restrict__ order) {
    pdl_prologue();
    __shared__ uint32_t s_warp[kTileScanThreads / 32];
    __shared__ uint32_t s_total;
    __shared__ uint32_t s_off[1024], s_loc[1024];
    const uint32_t t = threadIdx.x;
    s_loc[t] = 0;
    s_off[t] = block_exclusive_1024(counters->order_hist[t], s_warp, &s_total);  // bucket offsets
    const uint32_t i = blockIdx.x * kTileScanThreads + t;
    uint32_t bucket = 0, rank = 0;
    if (i < ntiles) {
        const uint4 sc = reinterpret_cast<const uint4*>(cnt)[i];
        bucket = 1023u - min(sc.x + sc.y + sc.z + sc.w, 1023u);
        rank = atomicAdd(&s_loc[bucket], 1u);
    }
    __syncthreads();
    // one range per non-empty bucket of this CTA
    if (s_loc[t]) s_loc[t] = s_off[t] + atomicAdd(&counters->order_cur[t], s_loc[t]);
    __syncthreads();
    if (i < ntiles) order[s_loc[bucket] + rank] = i;
}

void prepare_status(Ctx* c, uint32_t tiles) {
    const size_t need = static_cast<size_t>(tiles) + 1;
    if (c->scan_status_cap < need) {
        if (c->scan_status) cudaFree(c->scan_status);
        BSG_CUDA(cudaMalloc(&c->scan_status, 2 * need * sizeof(unsigned long long)));
        BSG_CUDA(cudaMemsetAsync(c->scan_status, 0, 2 * need * sizeof(unsigned long long), c->stream));  // epoch 0 is never used
        c->scan_status_cap = 2 * need;
    }
}

}  // namespace

Lookback next_lookback(Ctx* c, int which, uint32_t grid) {
    if (!c->lb_ticket) {
        BSG_CUDA(cudaMalloc(&c->lb_ticket, 2 * sizeof(unsigned long long)));
        BSG_CUDA(cudaMemsetAsync(c->lb_ticket, 0, 2 * sizeof(unsigned long long), c->stream));
        c->lb_next[0] = c->lb_next[1] = 0;
    }
    c->lb_epoch = (c->lb_epoch + 1) & 0x3fffffffu;
    if (c->lb_epoch == 0) c->lb_epoch = 1;
    Lookback lb{c->lb_ticket + which, c->lb_next[which], c->lb_epoch};
    c->lb_next[which] += grid;
    return lb;
}

void wait_mailbox(Ctx* c, const volatile uint32_t* seq_word, uint32_t seq) {
    for (uint32_t it = 1;; ++it) {
        if (*seq_word == seq) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return;
        }
        if ((it & 255u) == 0) {  // a failed or finished stream never writes it
            const cudaError_t e = cudaStreamQuery(c->stream);
            if (e == cudaSuccess) {
                if (*seq_word == seq) {
                    std::atomic_thread_fence(std::memory_order_acquire);
                    return;
                }
                throw Error{BSG_ERR_CUDA, "stream completed without writing the mailbox"};
            }
            if (e != cudaErrorNotReady) BSG_CUDA(e);
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#elif defined(__aarch64__)
        asm volatile("yield");
#endif
    }
}

void scan_exclusive_u32(Ctx* c, const uint32_t* in, const uint32_t* gather_idx, uint32_t* out, uint32_t n,
                        uint32_t* total_dev, const Publish& pub) {
    if (n == 0) {
        BSG_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), c->stream));
        if (pub.seq_word) throw Error{BSG_ERR_STATE, "empty scan cannot publish"};
        return;
    }
    const uint32_t tiles = (n + kScanTile - 1) / kScanTile;
    prepare_status(c, tiles);
    const Lookback lb = next_lookback(c, 0, tiles);
    launch_pdl(c->stream, tiles, kScanThreads, 0, scan_kernel<0>, in, gather_idx, out, n, c->scan_status, lb, pub, total_dev,
                                                          nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, 0,
                                                          nullptr);
    BSG_LAUNCHED(c);
}

void compact_visible(Ctx* c, uint32_t n, bool key32, const Publish& pub) {
    if (n == 0) {
        BSG_CUDA(cudaMemsetAsync(&c->counters->visible, 0, sizeof(uint32_t), c->stream));
        if (pub.seq_word) throw Error{BSG_ERR_STATE, "empty compaction cannot publish"};
        return;
    }
    const uint32_t tiles = (n + kScanTile - 1) / kScanTile;
    prepare_status(c, tiles);
    const Lookback lb = next_lookback(c, 0, tiles);
    if (key32)
        launch_pdl(c->stream, tiles, kScanThreads, 0, scan_kernel<2>, c->tiles, nullptr, c->vis_rows, n, c->scan_status, lb, pub,
                                                              &c->counters->visible, c->depth_key, c->vkey[0],
                                                              c->counters, c->vrow[0], &c->counters->depth_hist[0][0], 0,
                                                              c->vis_mask, static_cast<uint32_t>(c->cap / 32),
                                                              c->vis_prefix);
    else
        launch_pdl(c->stream, tiles, kScanThreads, 0, scan_kernel<1>, c->tiles, nullptr, c->vis_rows, n, c->scan_status, lb, pub,
                                                              &c->counters->visible, c->depth_key, c->vkey[0],
                                                              c->counters, c->vrow[0], &c->counters->depth_hist[0][0], 0,
                                                              c->vis_mask, static_cast<uint32_t>(c->cap / 32),
                                                              c->vis_prefix);
    BSG_LAUNCHED(c);
}

void compact_visible_mask(Ctx* c, uint32_t n, const Publish& pub) {
    const uint32_t nwords = (n + 31) / 32;
    const uint32_t tiles = std::max<uint32_t>(1, (nwords + kMaskTile - 1) / kMaskTile);
    prepare_status(c, tiles);
    const Lookback lb = next_lookback(c, 0, tiles);
    launch_pdl(c->stream, tiles, kScanThreads, 0, compact_mask_kernel, c->vis_mask, nwords, c->scan_status, lb, pub,
               &c->counters->visible, c->vis_rows);
    BSG_LAUNCHED(c);
}

void launch_tile_scan_multi(Ctx* c, uint32_t ntiles, uint32_t seq) {
    const uint32_t grid = std::max<uint32_t>(1, (ntiles + kTileScanThreads - 1) / kTileScanThreads);
    if (c->tile_scan_used) {  // a second scan this step (the emission re-run): its accumulators afresh
        BSG_CUDA(cudaMemsetAsync(&c->counters->order_hist[0], 0,
                                 offsetof(StepCounters, pad4) - offsetof(StepCounters, order_hist), c->stream));
        BSG_CUDA(cudaMemsetAsync(&c->counters->pairs_wide, 0, sizeof(unsigned long long), c->stream));
    }
    c->tile_scan_used = true;
    prepare_status(c, grid);
    const Lookback lb = next_lookback(c, 0, grid);
    launch_pdl(c->stream, grid, kTileScanThreads, 0, tile_scan_a_kernel, c->tile_cnt, ntiles, c->ranges, c->tile_cur,
               c->scan_status, lb, c->counters, c->mbox, seq);
    BSG_LAUNCHED(c);
    launch_pdl(c->stream, grid, kTileScanThreads, 0, tile_scan_b_kernel, c->tile_cnt, ntiles, c->counters,
               c->tile_order);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
