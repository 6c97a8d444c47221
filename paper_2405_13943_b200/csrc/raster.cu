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

namespace bsg {
namespace {

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
                                                         uint32_t pcap, uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_hist[2 * 256];
    for (int k = threadIdx.x; k < 512; k += blockDim.x) s_hist[k] = 0;
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
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t k = pkey[i];
    if (i == 0 || pkey[i - 1] != k) ranges[k].x = i;
    if (i == P - 1 || pkey[i + 1] != k) ranges[k].y = i + 1;
}

// K6: one CTA per 16x16 tile, one thread per pixel; splat records staged in
// shared memory 256 at a time. renderer.cpp:160-181 semantics: per pixel,
// contributors are the splats whose rect contains it, in (depth, index) order;
// break before compositing once T < stop; alpha = min(o g, clamp); no 1/255 skip.
__global__ __launch_bounds__(kTileThreads) void blend_fwd_kernel(const uint2* __restrict__ ranges,
                                                                 const uint32_t* __restrict__ pval,
                                                                 const float4* __restrict__ rec, int W, int H,
                                                                 int tiles_x, double tstop, float aclamp,
                                                                 double aclamp_d, float bg0,
                                                                 float bg1, float bg2, float* __restrict__ out_rgb,
                                                                 float* __restrict__ out_T,
                                                                 uint32_t* __restrict__ out_n,
                                                                 uint32_t* __restrict__ out_last) {
    __shared__ float4 s_a[kTileThreads], s_b[kTileThreads], s_c[kTileThreads];
    const int tile = blockIdx.x;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x % kTile);
    const int py = (tile / tiles_x) * kTile + (threadIdx.x / kTile);
    const bool inside = px < W && py < H;
    const uint2 range = ranges[tile];
    // The stop decision tracks T in FP64 like the reference: stacked clamped
    // splats give T = (1 - 0.99)^k exactly at the 1e-4 threshold (renderer
    // KAT test_renderer.cpp:272-282), which FP32 would cross one splat early.
    // Colour accumulation stays FP32.
    float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
    double Td = 1.0;
    const double oma_clamp = 1.0 - static_cast<double>(aclamp_d);
    uint32_t n = 0, last = 0;
    bool done = !inside;
    const float fx = static_cast<float>(px), fy = static_cast<float>(py);
    for (uint32_t start = range.x; start < range.y; start += kTileThreads) {
        if (__syncthreads_count(done) == kTileThreads) break;
        const uint32_t idx = start + threadIdx.x;
        if (idx < range.y) {
            const size_t r = 3 * static_cast<size_t>(pval[idx]);
            s_a[threadIdx.x] = rec[r];
            s_b[threadIdx.x] = rec[r + 1];
            s_c[threadIdx.x] = rec[r + 2];
        }
        __syncthreads();
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kTileThreads), range.y - start));
        for (int j = 0; !done && j < cnt; ++j) {
            const float4 c = s_c[j];
            int x0, x1, y0, y1;
            unpack_rect(c, x0, x1, y0, y1);
            if (px < x0 || px > x1 || py < y0 || py > y1) continue;
            if (Td < tstop) {
                done = true;
                break;
            }
            const float4 a = s_a[j], b = s_b[j];
            const float dx = fx - a.x, dy = fy - a.y;
            const float q = dx * (a.z * dx + a.w * dy) + dy * (a.w * dx + b.x * dy);
            const float g = __expf(-0.5f * q);
            const float og = b.y * g;
            // no float lies in [0.99, float(0.99)), so this is the FP64 clamp test
            const bool clamped = og >= aclamp;
            const float alpha = clamped ? aclamp : og;
            const float w = alpha * T;
            c0 += b.z * w;
            c1 += b.w * w;
            c2 += c.x * w;
            T *= 1.f - alpha;
            Td *= clamped ? oma_clamp : static_cast<double>(1.f - og);  // 1 - og exact for og >= 0.5
            ++n;
            last = start - range.x + j + 1;
        }
    }
    if (inside) {
        const size_t p = static_cast<size_t>(py) * W + px;
        out_rgb[3 * p + 0] = c0 + T * bg0;
        out_rgb[3 * p + 1] = c1 + T * bg1;
        out_rgb[3 * p + 2] = c2 + T * bg2;
        out_T[p] = static_cast<float>(Td);
        out_n[p] = n;
        out_last[p] = last;
    }
}

// Transpose-reduce of 16 per-lane values across a warp in 8+4+2+1+1 = 16
// shuffles (instead of 16 x 5): at each halving step a lane keeps one half
// of its values and receives the partner's copy of that half. On return,
// lane l holds the full warp sum of value index ((l >> 1) & 15) bit-reversed
// per the step order; `reduced_index` gives the mapping.
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
    const bool h16 = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float send = h16 ? v[k] : v[k + 8];
        const float keep = h16 ? v[k + 8] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    const bool h8 = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = h8 ? v[k] : v[k + 4];
        const float keep = h8 ? v[k + 4] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const bool h4 = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = h4 ? v[k] : v[k + 2];
        const float keep = h4 ? v[k + 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const bool h2 = lane & 2;
    {
        const float send = h2 ? v[0] : v[1];
        const float keep = h2 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Value index owned by `lane` after transpose_reduce16.
__device__ __forceinline__ int reduced_index(int lane) {
    return ((lane & 16) ? 8 : 0) + ((lane & 8) ? 4 : 0) + ((lane & 4) ? 2 : 0) + ((lane & 2) ? 1 : 0);
}

// K8: reverse traversal (renderer.cpp:274-311). Each pixel rewinds exactly
// the contributors it composited (T recovered by division, 1-alpha >= 0.01);
// the per-splat image-space gradients of the 32 pixels of a warp are reduced
// with shuffles before one set of global vector atomics per warp.
__global__ __launch_bounds__(kTileThreads) void blend_bwd_kernel(const uint2* __restrict__ ranges,
                                                                 const uint32_t* __restrict__ pval,
                                                                 const float4* __restrict__ rec, int W, int H,
                                                                 int tiles_x, float aclamp, float bg0, float bg1,
                                                                 float bg2, const float* __restrict__ in_T,
                                                                 const uint32_t* __restrict__ in_last,
                                                                 const float* __restrict__ dl_dc,
                                                                 float4* __restrict__ g2d) {
    __shared__ float4 s_a[kTileThreads], s_b[kTileThreads], s_c[kTileThreads];
    __shared__ uint32_t s_row[kTileThreads];
    __shared__ uint32_t s_max;
    const int tile = blockIdx.x;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x % kTile);
    const int py = (tile / tiles_x) * kTile + (threadIdx.x / kTile);
    const bool inside = px < W && py < H;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31;
    uint32_t my_last = 0;
    float T = 1.f, d0 = 0.f, d1 = 0.f, d2 = 0.f;
    if (inside) {
        const size_t p = static_cast<size_t>(py) * W + px;
        my_last = in_last[p];
        T = in_T[p];
        d0 = dl_dc[3 * p];
        d1 = dl_dc[3 * p + 1];
        d2 = dl_dc[3 * p + 2];
    }
    float s0 = T * bg0, s1 = T * bg1, s2 = T * bg2;  // suffix: contributions behind
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    // warp max then one shared atomic per warp
    uint32_t wm = my_last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (lane == 0) atomicMax(&s_max, wm);
    __syncthreads();
    const uint32_t max_last = s_max;
    const float fx = static_cast<float>(px), fy = static_cast<float>(py);
    for (int64_t end = max_last; end > 0; end -= kTileThreads) {
        const int64_t start = end - kTileThreads > 0 ? end - kTileThreads : 0;
        __syncthreads();
        const int64_t li = start + threadIdx.x;
        if (li < end) {
            const uint32_t row = pval[range.x + li];
            const size_t r = 3 * static_cast<size_t>(row);
            s_a[threadIdx.x] = rec[r];
            s_b[threadIdx.x] = rec[r + 1];
            s_c[threadIdx.x] = rec[r + 2];
            s_row[threadIdx.x] = row;
        }
        __syncthreads();
        for (int64_t j = end - 1; j >= start; --j) {
            const int sj = static_cast<int>(j - start);
            const float4 c = s_c[sj];
            int x0, x1, y0, y1;
            unpack_rect(c, x0, x1, y0, y1);
            const bool contrib = static_cast<uint32_t>(j) < my_last && px >= x0 && px <= x1 && py >= y0 && py <= y1;
            float gmx = 0.f, gmy = 0.f, gc00 = 0.f, gc01 = 0.f, gc11 = 0.f, gr = 0.f, gg = 0.f, gb = 0.f, go = 0.f;
            if (contrib) {
                const float4 a = s_a[sj], b = s_b[sj];
                const float dx = fx - a.x, dy = fy - a.y;
                const float mdx = a.z * dx + a.w * dy, mdy = a.w * dx + b.x * dy;
                const float q = dx * mdx + dy * mdy;
                const float g = __expf(-0.5f * q);
                const float og = b.y * g;
                const float alpha = fminf(og, aclamp);
                const float oma = 1.f - alpha;
                const float inv = 1.f / oma;
                const float Tb = T * inv;
                const float at = alpha * Tb;
                gr = d0 * at;
                gg = d1 * at;
                gb = d2 * at;
                const float dlda = (d0 * (b.z * Tb - s0 * inv) + d1 * (b.w * Tb - s1 * inv)) + d2 * (c.x * Tb - s2 * inv);
                if (og < aclamp) {
                    const float dl_dg = dlda * b.y;
                    const float k = dl_dg * g;
                    gmx = k * mdx;
                    gmy = k * mdy;
                    const float h = 0.5f * k;
                    gc00 = h * (mdx * mdx);
                    gc01 = h * (mdx * mdy);
                    gc11 = h * (mdy * mdy);
                    go = dlda * g;
                }
                s0 += b.z * at;
                s1 += b.w * at;
                s2 += c.x * at;
                T = Tb;
            }
            const unsigned mask = __ballot_sync(0xffffffffu, contrib);
            if (mask == 0) continue;
            float* dst = reinterpret_cast<float*>(g2d + 3 * static_cast<size_t>(s_row[sj]));
            if (__popc(mask) <= 2) {
                // one or two contributing pixels: direct atomics are cheaper than a reduction
                if (contrib) {
                    atomicAdd(reinterpret_cast<float4*>(dst), make_float4(gmx, gmy, gc00, gc01));
                    atomicAdd(reinterpret_cast<float4*>(dst) + 1, make_float4(gc11, gr, gg, gb));
                    atomicAdd(dst + 8, go);
                }
            } else {
                float vals[16] = {gmx, gmy, gc00, gc01, gc11, gr, gg, gb, go, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                const float r = transpose_reduce16(vals, lane);
                const int idx = reduced_index(lane);
                if ((lane & 1) == 0 && idx < 9) atomicAdd(dst + idx, r);
            }
        }
    }
}

}  // namespace

void launch_pairs(Ctx* c, const DevCam& cam, uint32_t V) {
    if (V == 0) return;
    emit_pairs_kernel<<<(V + 255) / 256, 256, 0, c->stream>>>(c->vrow[c->depth_sorted], c->poff, c->rec, V, cam.tiles_x,
                                                              c->pkey[0], c->pval[0], static_cast<uint32_t>(c->pcap),
                                                              &c->counters->tile_hist[0][0]);
    BSG_LAUNCHED(c);
}

void launch_ranges(Ctx* c, const DevCam& cam, uint32_t P) {
    const size_t ntiles = static_cast<size_t>(cam.tiles_x) * cam.tiles_y;
    BSG_CUDA(cudaMemsetAsync(c->ranges, 0, ntiles * sizeof(uint2), c->stream));
    if (P == 0) return;
    ranges_kernel<<<(P + 255) / 256, 256, 0, c->stream>>>(c->pkey[c->pairs_sorted], P, c->ranges);
    BSG_LAUNCHED(c);
}

void launch_blend_fwd(Ctx* c, const DevCam& cam, const DevRender& rc) {
    const int ntiles = cam.tiles_x * cam.tiles_y;
    blend_fwd_kernel<<<ntiles, kTileThreads, 0, c->stream>>>(
        c->ranges, c->pval[c->pairs_sorted], c->rec, cam.W, cam.H, cam.tiles_x, rc.tstop,
        static_cast<float>(rc.alpha_clamp), rc.alpha_clamp, rc.bg[0], rc.bg[1], rc.bg[2], c->out_rgb, c->out_T,
        c->out_n, c->out_last);
    BSG_LAUNCHED(c);
}

void launch_blend_bwd(Ctx* c, const DevCam& cam, const DevRender& rc) {
    const int ntiles = cam.tiles_x * cam.tiles_y;
    blend_bwd_kernel<<<ntiles, kTileThreads, 0, c->stream>>>(
        c->ranges, c->pval[c->pairs_sorted], c->rec, cam.W, cam.H, cam.tiles_x, static_cast<float>(rc.alpha_clamp),
        rc.bg[0], rc.bg[1], rc.bg[2], c->out_T, c->out_last, c->dl_dc, c->g2d);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
