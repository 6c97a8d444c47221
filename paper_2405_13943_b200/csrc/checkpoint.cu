// GSPL checkpoint payload on the device (scene_io.cpp:48-59). The float part
// of the section is five row-interleaved arrays -- positions [n][3],
// rotations [n][4], log-scales [n][3], features [n][F], opacity logits [n] --
// gathered from the row-major device store (row_stride / pslot) group by group.
// One streaming kernel writes it in section order (coalesced stores, reads of
// w consecutive components of consecutive rows); the host prepends the count,
// width and ids. HBM-bound: 4 D n bytes read, 4 D n written.
#include "bsg_internal.cuh"

#include <algorithm>

namespace bsg {
namespace {

__global__ __launch_bounds__(256) void gspl_floats_kernel(const float* __restrict__ x, size_t cap, uint32_t n, int fd,
                                                          float* __restrict__ out) {
    const uint64_t total = static_cast<uint64_t>(11 + fd) * n;
    // group starts (in output floats) and widths: pos 3, rot 4, ls 3, feat fd, op 1
    const uint64_t s1 = 3ull * n, s2 = 7ull * n, s3 = 10ull * n, s4 = static_cast<uint64_t>(10 + fd) * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t local;
        int w, c0;
        if (e < s1) { local = e; w = 3; c0 = kPos; }
        else if (e < s2) { local = e - s1; w = 4; c0 = kRot; }
        else if (e < s3) { local = e - s2; w = 3; c0 = kLs; }
        else if (e < s4) { local = e - s3; w = fd; c0 = kFeat; }
        else { local = e - s4; w = 1; c0 = op_comp(fd); }
        const uint64_t row = local / static_cast<uint64_t>(w);
        const int k = static_cast<int>(local - row * static_cast<uint64_t>(w));
        out[e] = x[pidx(row, c0 + k, fd)];
    }
}

}  // namespace

void launch_gspl_floats(Ctx* c, float* out) {
    if (c->n == 0) return;
    const uint64_t total = static_cast<uint64_t>(11 + c->fd) * c->n;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
    materialize(c);
    gspl_floats_kernel<<<grid, 256, 0, c->stream>>>(c->x, c->cap, static_cast<uint32_t>(c->n), c->fd, out);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
