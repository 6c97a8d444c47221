// Host-side block planner: the recursive longer-axis bipartition and the
// expanded-box assignment (splitter.cpp:48-201) plus the shard/owner
// bookkeeping of plan_cluster (runtime.cpp:265-305), and the compact slot
// index the consensus reduction runs over. Runs once per run on the CPU; its
// outputs (block membership, shared sets) are an integer parity contract with
// the reference, so every comparison below is the reference's.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bsgpu.h"

namespace {

struct Box {
    double mn[3], mx[3];
    bool contains(const double* p) const {
        for (int a = 0; a < 3; ++a)
            if (!(p[a] >= mn[a])) return false;
        for (int a = 0; a < 3; ++a)
            if (!(p[a] <= mx[a])) return false;
        return true;
    }
    double distance(const double* p) const {  // splitter.hpp:24-27
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = std::max(std::max(mn[a] - p[a], p[a] - mx[a]), 0.0);
        return std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    }
};

Box tight(const double* pos, const std::vector<size_t>& idx) {
    Box b;
    for (int a = 0; a < 3; ++a) b.mn[a] = b.mx[a] = pos[3 * idx[0] + a];
    for (size_t i : idx)
        for (int a = 0; a < 3; ++a) {
            b.mn[a] = std::min(b.mn[a], pos[3 * i + a]);
            b.mx[a] = std::max(b.mx[a], pos[3 * i + a]);
        }
    return b;
}

struct Cell {
    Box box;
    std::vector<size_t> idx;
};

}  // namespace

struct bsg_plan {
    uint32_t k = 0;
    std::vector<Box> core, expanded;
    std::vector<std::vector<uint64_t>> block_ids;  // ascending
    std::vector<std::vector<uint32_t>> block_views;
    std::vector<uint64_t> shared_ids;              // ascending, >= 2 owners
    std::vector<uint32_t> shared_owner_count;
    std::vector<uint32_t> shared_first_owner;
};

namespace {
thread_local std::string g_plan_err;

template <typename F>
int guarded_plan(F&& f) {
    try {
        f();
        return BSG_OK;
    } catch (const std::invalid_argument& e) {
        g_plan_err = e.what();
        return BSG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_plan_err = e.what();
        return BSG_ERR_STATE;
    }
}
}  // namespace

extern "C" {

const char* bsg_plan_last_error(void) { return g_plan_err.c_str(); }

int bsg_plan_create(size_t n, const uint64_t* ids, const double* pos, size_t n_views, const double* view_centers,
                    uint32_t k, double scale, int vertical_axis, int midpoint_plane, bsg_plan** out) {
    return guarded_plan([&] {
        if (!out) throw std::invalid_argument("null output");
        if (k < 1) throw std::invalid_argument("k must be at least 1");
        if (n == 0) throw std::invalid_argument("empty point set");
        if (k > n) throw std::invalid_argument("over-partitioned");
        if (scale < 1.0) throw std::invalid_argument("expansion scale must be >= 1");
        for (size_t i = 1; i < n; ++i)
            if (ids[i] <= ids[i - 1]) throw std::invalid_argument("initial cloud ill-formed");
        const int va = vertical_axis;
        auto pick_axis = [va](const Box& b) {  // splitter.cpp:32-44
            int best = -1;
            double best_len = -1.0;
            for (int a = 0; a < 3; ++a) {
                if (a == va) continue;
                const double len = b.mx[a] - b.mn[a];
                if (len > best_len) {
                    best_len = len;
                    best = a;
                }
            }
            return best;
        };
        // split_recursive (splitter.cpp:48-96)
        std::vector<Cell> cells(1);
        cells[0].idx.resize(n);
        std::iota(cells[0].idx.begin(), cells[0].idx.end(), size_t{0});
        cells[0].box = tight(pos, cells[0].idx);
        while (cells.size() < k) {
            size_t target = 0;
            for (size_t c = 1; c < cells.size(); ++c)
                if (cells[c].idx.size() > cells[target].idx.size()) target = c;
            Cell cell = std::move(cells[target]);
            const int axis = pick_axis(cell.box);
            std::vector<size_t>& idx = cell.idx;
            auto less = [&](size_t a, size_t b) {
                if (pos[3 * a + axis] != pos[3 * b + axis]) return pos[3 * a + axis] < pos[3 * b + axis];
                return a < b;
            };
            size_t cut;
            if (midpoint_plane) {
                std::sort(idx.begin(), idx.end(), less);
                const double plane = 0.5 * (cell.box.mn[axis] + cell.box.mx[axis]);
                cut = static_cast<size_t>(std::lower_bound(idx.begin(), idx.end(), plane,
                                                           [&](size_t a, double v) { return pos[3 * a + axis] < v; }) -
                                          idx.begin());
                cut = std::clamp<size_t>(cut, 1, idx.size() - 1);
            } else {
                // The median cut of the (coordinate, index) order only needs the
                // partition, not the full sort: same sets as the reference.
                cut = idx.size() / 2;
                std::nth_element(idx.begin(), idx.begin() + static_cast<ptrdiff_t>(cut), idx.end(), less);
            }
            Cell left, right;
            left.idx.assign(idx.begin(), idx.begin() + static_cast<ptrdiff_t>(cut));
            right.idx.assign(idx.begin() + static_cast<ptrdiff_t>(cut), idx.end());
            left.box = tight(pos, left.idx);
            right.box = tight(pos, right.idx);
            cells[target] = std::move(left);
            cells.push_back(std::move(right));
        }
        auto* p = new bsg_plan();
        p->k = k;
        // expand_and_assign (splitter.cpp:98-201); the points are the Gaussian
        // positions themselves (runtime.cpp:279-284).
        double vmin = std::numeric_limits<double>::infinity(), vmax = -vmin;
        for (size_t i = 0; i < n; ++i) {
            vmin = std::min(vmin, pos[3 * i + va]);
            vmax = std::max(vmax, pos[3 * i + va]);
        }
        for (const Cell& c : cells) {
            p->core.push_back(c.box);
            Box e = c.box;
            for (int a = 0; a < 3; ++a) {
                if (a == va) continue;
                const double ctr = 0.5 * (c.box.mn[a] + c.box.mx[a]);
                const double half = 0.5 * (c.box.mx[a] - c.box.mn[a]) * scale;
                e.mn[a] = std::min(c.box.mn[a], ctr - half);
                e.mx[a] = std::max(c.box.mx[a], ctr + half);
            }
            e.mn[va] = vmin;
            e.mx[va] = vmax;
            p->expanded.push_back(e);
        }
        p->block_ids.resize(k);
        p->block_views.resize(k);
        std::vector<uint32_t> who;
        for (size_t i = 0; i < n; ++i) {
            const double* q = pos + 3 * i;
            who.clear();
            for (uint32_t b = 0; b < k; ++b)
                if (p->expanded[b].contains(q)) who.push_back(b);
            if (who.empty()) {
                uint32_t best = 0;
                double best_d = p->expanded[0].distance(q);
                for (uint32_t b = 1; b < k; ++b) {
                    const double d = p->expanded[b].distance(q);
                    if (d < best_d) {
                        best_d = d;
                        best = b;
                    }
                }
                who.push_back(best);
            }
            for (uint32_t b : who) p->block_ids[b].push_back(ids[i]);
            if (who.size() >= 2) {
                p->shared_ids.push_back(ids[i]);
                p->shared_owner_count.push_back(static_cast<uint32_t>(who.size()));
                p->shared_first_owner.push_back(who[0]);
            }
        }
        for (size_t v = 0; v < n_views; ++v) {
            const double* c = view_centers + 3 * v;
            bool placed = false;
            for (uint32_t b = 0; b < k; ++b)
                if (p->expanded[b].contains(c)) {
                    p->block_views[b].push_back(static_cast<uint32_t>(v));
                    placed = true;
                }
            if (!placed) {
                uint32_t best = 0;
                double best_d = 0;
                for (uint32_t b = 0; b < k; ++b) {
                    double e[3];
                    for (int a = 0; a < 3; ++a) e[a] = 0.5 * (p->expanded[b].mn[a] + p->expanded[b].mx[a]) - c[a];
                    const double d = (e[0] * e[0] + e[1] * e[1]) + e[2] * e[2];
                    if (b == 0 || d < best_d) {
                        best_d = d;
                        best = b;
                    }
                }
                p->block_views[best].push_back(static_cast<uint32_t>(v));
            }
        }
        *out = p;
    });
}

void bsg_plan_destroy(bsg_plan* p) { delete p; }

int bsg_plan_block_sizes(const bsg_plan* p, uint32_t b, size_t* n_gaussians, size_t* n_views) {
    return guarded_plan([&] {
        if (!p || b >= p->k) throw std::invalid_argument("block id out of range");
        if (n_gaussians) *n_gaussians = p->block_ids[b].size();
        if (n_views) *n_views = p->block_views[b].size();
    });
}

int bsg_plan_block(const bsg_plan* p, uint32_t b, uint64_t* ids, uint32_t* views) {
    return guarded_plan([&] {
        if (!p || b >= p->k) throw std::invalid_argument("block id out of range");
        if (ids) std::copy(p->block_ids[b].begin(), p->block_ids[b].end(), ids);
        if (views) std::copy(p->block_views[b].begin(), p->block_views[b].end(), views);
    });
}

int bsg_plan_boxes(const bsg_plan* p, double* core_min, double* core_max, double* exp_min, double* exp_max) {
    return guarded_plan([&] {
        if (!p) throw std::invalid_argument("null plan");
        for (uint32_t b = 0; b < p->k; ++b)
            for (int a = 0; a < 3; ++a) {
                if (core_min) core_min[3 * b + a] = p->core[b].mn[a];
                if (core_max) core_max[3 * b + a] = p->core[b].mx[a];
                if (exp_min) exp_min[3 * b + a] = p->expanded[b].mn[a];
                if (exp_max) exp_max[3 * b + a] = p->expanded[b].mx[a];
            }
    });
}

size_t bsg_plan_shared_count(const bsg_plan* p) { return p ? p->shared_ids.size() : 0; }

// Global consensus slots: slot s = s-th shared id in ascending order.
int bsg_plan_shared(const bsg_plan* p, uint64_t* ids, uint32_t* owner_count, uint32_t* first_owner) {
    return guarded_plan([&] {
        if (!p) throw std::invalid_argument("null plan");
        if (ids) std::copy(p->shared_ids.begin(), p->shared_ids.end(), ids);
        if (owner_count) std::copy(p->shared_owner_count.begin(), p->shared_owner_count.end(), owner_count);
        if (first_owner) std::copy(p->shared_first_owner.begin(), p->shared_first_owner.end(), first_owner);
    });
}

// This block's anchor rows for bsg_set_shared: rows into the block's cloud,
// slots into the global slot table, first-owner flags.
int bsg_plan_block_shared(const bsg_plan* p, uint32_t b, size_t* n_out, uint32_t* rows, uint32_t* slots,
                          uint8_t* first) {
    return guarded_plan([&] {
        if (!p || b >= p->k) throw std::invalid_argument("block id out of range");
        const std::vector<uint64_t>& mine = p->block_ids[b];
        size_t cnt = 0;
        size_t i = 0;
        for (size_t s = 0; s < p->shared_ids.size(); ++s) {
            const uint64_t id = p->shared_ids[s];
            while (i < mine.size() && mine[i] < id) ++i;
            if (i < mine.size() && mine[i] == id) {
                if (rows) rows[cnt] = static_cast<uint32_t>(i);
                if (slots) slots[cnt] = static_cast<uint32_t>(s);
                if (first) first[cnt] = p->shared_first_owner[s] == b ? 1 : 0;
                ++cnt;
            }
        }
        if (n_out) *n_out = cnt;
    });
}

}  // extern "C"
