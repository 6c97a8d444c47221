// Master-round ownership bookkeeping on the device (the
// reference's runtime.cpp:490-518 over a std::map of every id's owners).
//
// Only ids in the consensus slot table can change class: a non-shared id has
// one owner, so its removal kills it, and new rows are born single-owner
// (runtime.cpp:514-517). The table is therefore the slot table itself -- the
// shared ids (ascending, as the slots are numbered) and a bitmask of their
// owning blocks (K <= 32) -- resident on the master block's device. A round
// binary-searches every removed id into it (one thread per id), clears the
// removing block's bit, classifies each touched slot by its owner counts
// before / after (reset: still >= 2 owners; unshared: 1; dead: 0), compacts
// the table to the slots that keep >= 2 owners, and returns only the touched
// slots (ascending) -- O(removed + S / threads) on the device, O(touched) to
// the host, no host map.
#include "bsg_internal.cuh"

namespace bsg {
namespace {

constexpr int kOwnThreads = 256;
constexpr int kOwnScanItems = 4;  // slots per thread in the scan
constexpr int kOwnChunk = kOwnThreads * kOwnScanItems;

__global__ __launch_bounds__(kOwnThreads) void own_mark_kernel(const uint64_t* __restrict__ in_ids,
                                                              const uint32_t* __restrict__ in_blk, uint32_t m,
                                                              const uint64_t* __restrict__ ids, uint32_t n,
                                                              uint32_t* __restrict__ rm,
                                                              uint8_t* __restrict__ found) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t id = in_ids[i];
    BSG_DASSERT(in_blk[i] < 32);
    uint32_t lo = 0, hi = n;  // first slot with ids[slot] >= id
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ids[mid] < id)
            lo = mid + 1;
        else
            hi = mid;
    }
    const bool hit = lo < n && ids[lo] == id;
    found[i] = hit ? 1 : 0;
    if (hit) atomicOr(&rm[lo], 1u << in_blk[i]);
}

// Class of a slot this round: 0 untouched, 1 reset (>= 2 owners remain),
// 2 unshared (1 remains), 3 dead (none). keep = >= 2 owners remain.
__device__ __forceinline__ uint32_t own_class(uint32_t r, uint32_t now) {
    if (!r) return 0;
    const int c = __popc(now);
    return c == 0 ? 3u : (c == 1 ? 2u : 1u);
}

// Per chunk of kOwnChunk slots: the number kept and the number touched.
__global__ __launch_bounds__(kOwnThreads) void own_count_kernel(const uint32_t* __restrict__ mask,
                                                               const uint32_t* __restrict__ rm, uint32_t n,
                                                               uint2* __restrict__ chunk_tot) {
    __shared__ uint32_t s_keep, s_touch;
    if (threadIdx.x == 0) {
        s_keep = 0;
        s_touch = 0;
    }
    __syncthreads();
    uint32_t keep = 0, touch = 0;
    const uint32_t base = blockIdx.x * kOwnChunk;
#pragma unroll
    for (int k = 0; k < kOwnScanItems; ++k) {
        const uint32_t s = base + k * kOwnThreads + threadIdx.x;
        if (s < n) {
            const uint32_t now = mask[s] & ~rm[s];
            keep += __popc(now) >= 2;
            touch += rm[s] != 0;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        keep += __shfl_xor_sync(0xffffffffu, keep, o);
        touch += __shfl_xor_sync(0xffffffffu, touch, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_keep, keep);
        atomicAdd(&s_touch, touch);
    }
    __syncthreads();
    if (threadIdx.x == 0) chunk_tot[blockIdx.x] = make_uint2(s_keep, s_touch);
}

// One CTA: exclusive scan of the chunk totals (both components) in place;
// the grand totals land in totals[0..1].
__global__ __launch_bounds__(1024) void own_scan_chunks_kernel(uint2* __restrict__ chunk_tot, uint32_t nchunks,
                                                               uint32_t* __restrict__ totals) {
    __shared__ uint2 s_warp[32];
    __shared__ uint2 s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = make_uint2(0, 0);
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nchunks; b0 += 1024) {
        const uint32_t i = b0 + threadIdx.x;
        const uint2 v = i < nchunks ? chunk_tot[i] : make_uint2(0, 0);
        uint2 inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, inc.x, o), b = __shfl_up_sync(0xffffffffu, inc.y, o);
            if (lane >= o) {
                inc.x += a;
                inc.y += b;
            }
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            uint2 w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t a = __shfl_up_sync(0xffffffffu, w.x, o), b = __shfl_up_sync(0xffffffffu, w.y, o);
                if (lane >= o) {
                    w.x += a;
                    w.y += b;
                }
            }
            s_warp[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const uint2 before = warp ? s_warp[warp - 1] : make_uint2(0, 0);
        const uint2 carry = s_carry;
        if (i < nchunks) chunk_tot[i] = make_uint2(carry.x + before.x + inc.x - v.x, carry.y + before.y + inc.y - v.y);
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = make_uint2(carry.x + before.x + inc.x, carry.y + before.y + inc.y);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        totals[0] = s_carry.x;
        totals[1] = s_carry.y;
    }
}

// Compaction of the kept slots into the other buffer (order preserved) and
// the touched slots' (slot, class, new mask) in slot order; clears rm.
__global__ __launch_bounds__(kOwnThreads) void own_compact_kernel(
    const uint64_t* __restrict__ ids, const uint32_t* __restrict__ mask, uint32_t* __restrict__ rm, uint32_t n,
    const uint2* __restrict__ chunk_off, uint64_t* __restrict__ ids_out, uint32_t* __restrict__ mask_out,
    uint32_t* __restrict__ t_slot, uint8_t* __restrict__ t_class, uint32_t* __restrict__ t_mask) {
    __shared__ uint32_t s_warp[2][kOwnThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = blockIdx.x * kOwnChunk;
    uint2 run = chunk_off[blockIdx.x];
    for (int k = 0; k < kOwnScanItems; ++k) {
        const uint32_t s = base + k * kOwnThreads + threadIdx.x;
        uint32_t now = 0, r = 0, m0 = 0;
        if (s < n) {
            m0 = mask[s];
            r = rm[s];
            now = m0 & ~r;
        }
        const bool keep = s < n && __popc(now) >= 2, touch = s < n && r != 0;
        const uint32_t bk = __ballot_sync(0xffffffffu, keep), bt = __ballot_sync(0xffffffffu, touch);
        if (lane == 0) {
            s_warp[0][warp] = __popc(bk);
            s_warp[1][warp] = __popc(bt);
        }
        __syncthreads();
        uint32_t ok = 0, ot = 0, tk = 0, tt = 0;
#pragma unroll
        for (int w = 0; w < kOwnThreads / 32; ++w) {
            if (w < warp) {
                ok += s_warp[0][w];
                ot += s_warp[1][w];
            }
            tk += s_warp[0][w];
            tt += s_warp[1][w];
        }
        const uint32_t lm = (1u << lane) - 1u;
        if (keep) {
            const uint32_t d = run.x + ok + __popc(bk & lm);
            ids_out[d] = ids[s];
            mask_out[d] = now;
        }
        if (touch) {
            const uint32_t d = run.y + ot + __popc(bt & lm);
            t_slot[d] = s;
            t_class[d] = static_cast<uint8_t>(own_class(r, now));
            t_mask[d] = now;
            rm[s] = 0;
        }
        run.x += tk;
        run.y += tt;
        __syncthreads();
    }
}

}  // namespace

void owners_alloc(OwnerTable* t, size_t n) {
    if (n <= t->cap) return;
    const size_t cap = std::max<size_t>(n, 1024);
    for (int k = 0; k < 2; ++k) {
        if (t->ids[k]) cudaFree(t->ids[k]);
        if (t->mask[k]) cudaFree(t->mask[k]);
        BSG_CUDA(cudaMalloc(&t->ids[k], cap * sizeof(uint64_t)));
        BSG_CUDA(cudaMalloc(&t->mask[k], cap * sizeof(uint32_t)));
    }
    if (t->rm) cudaFree(t->rm);
    if (t->chunk) cudaFree(t->chunk);
    BSG_CUDA(cudaMalloc(&t->rm, cap * sizeof(uint32_t)));
    BSG_CUDA(cudaMemset(t->rm, 0, cap * sizeof(uint32_t)));
    BSG_CUDA(cudaMalloc(&t->chunk, ((cap + kOwnChunk - 1) / kOwnChunk) * sizeof(uint2)));
    t->cap = cap;
}

// Runs one round's removals; returns the number of touched slots, whose
// (slot, class, mask) are in t->t_slot / t_class / t_mask (device), and leaves
// the compacted table current. found[i] (device) flags removed ids that were
// in the table.
uint32_t owners_round(OwnerTable* t, const uint64_t* d_in_ids, const uint32_t* d_in_blk, uint32_t m,
                      uint8_t* d_found) {
    const uint32_t n = t->n;
    if (m) {
        own_mark_kernel<<<(m + kOwnThreads - 1) / kOwnThreads, kOwnThreads, 0, t->stream>>>(
            d_in_ids, d_in_blk, m, t->ids[t->cur], n, t->rm, d_found);
        BSG_CUDA(cudaGetLastError());
    }
    if (n == 0) return 0;
    const uint32_t nchunks = (n + kOwnChunk - 1) / kOwnChunk;
    own_count_kernel<<<nchunks, kOwnThreads, 0, t->stream>>>(t->mask[t->cur], t->rm, n, t->chunk);
    own_scan_chunks_kernel<<<1, 1024, 0, t->stream>>>(t->chunk, nchunks, t->totals_dev);
    BSG_CUDA(cudaMemcpyAsync(t->totals_host, t->totals_dev, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, t->stream));
    BSG_CUDA(cudaStreamSynchronize(t->stream));
    const uint32_t kept = t->totals_host[0], touched = t->totals_host[1];
    if (touched > t->t_cap) {
        if (t->t_slot) cudaFree(t->t_slot);
        if (t->t_class) cudaFree(t->t_class);
        if (t->t_mask) cudaFree(t->t_mask);
        t->t_cap = std::max<size_t>(touched, 1024);
        BSG_CUDA(cudaMalloc(&t->t_slot, t->t_cap * sizeof(uint32_t)));
        BSG_CUDA(cudaMalloc(&t->t_class, t->t_cap));
        BSG_CUDA(cudaMalloc(&t->t_mask, t->t_cap * sizeof(uint32_t)));
    }
    if (touched == 0) return 0;
    own_compact_kernel<<<nchunks, kOwnThreads, 0, t->stream>>>(t->ids[t->cur], t->mask[t->cur], t->rm, n, t->chunk,
                                                               t->ids[1 - t->cur], t->mask[1 - t->cur], t->t_slot,
                                                               t->t_class, t->t_mask);
    BSG_CUDA(cudaGetLastError());
    t->cur = 1 - t->cur;
    t->n = kept;
    return touched;
}

}  // namespace bsg
