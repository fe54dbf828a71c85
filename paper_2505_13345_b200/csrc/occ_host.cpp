// occ_host.cpp — host-side collaboration-aware placement (stays on the CPU:
// it runs once per profiling window over an E x E table).
//
// normalize_graph   : collab.cpp:31-39 (counts / max edge; all-zero stays 0)
// reschedule_placement : placement.cpp:60-148, Alg. 1 — greedy clustering.
//   Bit-exact with the reference: the per-candidate means are accumulated in
//   member-list order and ties break to the lower expert index.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../../include/occult.h"

namespace occ {
occ_status host_fail(occ_status s, const char* msg);  // occ_capi.cu
}  // namespace occ

namespace {

// Mean collaboration of candidate `e` with a member list, summed in list order.
double mean_with(const double* p, int ne, const std::vector<int>& members, int e) {
    double sum = 0.0;
    for (int m : members) sum += p[static_cast<size_t>(m) * ne + e];
    return sum / static_cast<double>(members.size());
}

}  // namespace

extern "C" occ_status occ_normalize_graph(const int64_t* counts, int e, double* p) {
    if (!counts || !p || e < 1) return OCC_ERR_ARG;
    const size_t n = static_cast<size_t>(e) * e;
    int64_t mx = 0;
    for (size_t i = 0; i < n; ++i) mx = counts[i] > mx ? counts[i] : mx;
    for (size_t i = 0; i < n; ++i) p[i] = mx == 0 ? 0.0 : static_cast<double>(counts[i]) / static_cast<double>(mx);
    return OCC_OK;
}

extern "C" occ_status occ_reschedule_placement(const double* p, int ne, int nd, int32_t* out) {
    if (!p || !out) return OCC_ERR_ARG;
    if (nd < 1 || ne < 1 || ne % nd != 0) return OCC_ERR_CONFIG;
    const int per = ne / nd;
    std::vector<char> used(ne, 0);
    std::vector<int> assigned;  // every expert placed so far, in placement order
    assigned.reserve(ne);
    for (int d = 0; d < nd; ++d) {
        std::vector<int> dev;
        auto take = [&](int e) {
            dev.push_back(e);
            used[e] = 1;
            assigned.push_back(e);
        };
        if (d == 0) {
            if (ne == 1) {
                take(0);
            } else {
                // most collaborative pair: upper triangle, row-major, first maximum wins
                int bi = 0, bj = 1;
                double best = -1.0;
                for (int i = 0; i < ne; ++i)
                    for (int j = i + 1; j < ne; ++j) {
                        const double v = p[static_cast<size_t>(i) * ne + j];
                        if (v > best) { best = v; bi = i; bj = j; }
                    }
                take(bi);
                if (per >= 2) take(bj);
            }
        } else {
            // seed: the unused expert least collaborative with everything placed
            int pick = -1;
            double best = 0.0;
            for (int e = 0; e < ne; ++e) {
                if (used[e]) continue;
                const double s = mean_with(p, ne, assigned, e);
                if (pick < 0 || s < best) { best = s; pick = e; }
            }
            take(pick);
        }
        while (static_cast<int>(dev.size()) < per) {
            int pick = -1;
            double best = 0.0;
            for (int e = 0; e < ne; ++e) {
                if (used[e]) continue;
                const double s = mean_with(p, ne, dev, e);
                if (pick < 0 || s > best) { best = s; pick = e; }
            }
            take(pick);
        }
        for (int i = 0; i < per; ++i) out[d * per + i] = dev[i];
    }
    return OCC_OK;
}

// Layout of the two all-to-alls for EP rank `rank` given the all-gathered
// (source, destination) Sfd row counts C [nd x nd] (all_to_all_exchange,
// pipeline.cpp:125-176):
//   send to p  : this source's Sfd batch is device-major (BRIM0 counters,
//                pipeline.cpp:31-47), so the rows for p start at
//                sum_{d<p} C[rank][d] and number C[rank][p];
//   recv from p: the inbox is ordered (source asc, counter asc), so source p
//                lands at sum_{s<p} C[s][rank] and brings C[p][rank] rows.
// The return all-to-all uses the same four arrays with send/recv swapped.
extern "C" occ_status occ_exchange_layout(const int32_t* C, int nd, int rank, int64_t* send_off, int64_t* send_cnt,
                                          int64_t* recv_off, int64_t* recv_cnt) {
    if (!C || !send_off || !send_cnt || !recv_off || !recv_cnt) return OCC_ERR_ARG;
    if (nd < 1 || rank < 0 || rank >= nd) return OCC_ERR_CONFIG;
    int64_t so = 0, ro = 0;
    for (int p = 0; p < nd; ++p) {
        const int64_t sc = C[static_cast<size_t>(rank) * nd + p];
        const int64_t rc = C[static_cast<size_t>(p) * nd + rank];
        if (sc < 0 || rc < 0) return OCC_ERR_SHAPE;
        send_off[p] = so;
        send_cnt[p] = sc;
        recv_off[p] = ro;
        recv_cnt[p] = rc;
        so += sc;
        ro += rc;
    }
    return OCC_OK;
}

// ------------------------------------------------------- deterministic RNG
// rng.hpp:12-38: std::mt19937_64 (its output sequence is fixed by the C++
// standard) with the reference's own derived draws, so streams, synthetic
// inputs and traces are identical to the reference CLI's for the same seed.
struct occ_rng {
    std::mt19937_64 g;
    explicit occ_rng(uint64_t seed) : g(seed) {}
    double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }  // [0, 1)
    double between(double lo, double hi) { return lo + (hi - lo) * unit(); }
    int below(int n) {  // unbiased [0, n) by rejection above the largest multiple of n
        const uint64_t un = static_cast<uint64_t>(n);
        const uint64_t cut = UINT64_MAX - UINT64_MAX % un;
        uint64_t r = g();
        while (r >= cut) r = g();
        return static_cast<int>(r % un);
    }
};

extern "C" occ_status occ_rng_create(uint64_t seed, occ_rng** out) {
    if (!out) return occ::host_fail(OCC_ERR_ARG, "null argument");
    *out = new occ_rng(seed);
    return OCC_OK;
}

extern "C" void occ_rng_destroy(occ_rng* r) { delete r; }

extern "C" uint64_t occ_rng_next(occ_rng* r) { return r ? r->g() : 0; }

// random_matrix (core.cpp:54-58): row-major uniform [-1, 1), rounded through
// float for single precision.
extern "C" occ_status occ_rng_matrix(occ_rng* r, int rows, int cols, int single, double* out) {
    if (!r || (!out && rows > 0 && cols > 0)) return occ::host_fail(OCC_ERR_ARG, "null argument");
    if (rows < 0 || cols < 0) return occ::host_fail(OCC_ERR_SHAPE, "random_matrix: negative shape");
    const size_t n = static_cast<size_t>(rows) * cols;
    for (size_t i = 0; i < n; ++i) {
        const double v = r->between(-1.0, 1.0);
        out[i] = single ? static_cast<double>(static_cast<float>(v)) : v;
    }
    return OCC_OK;
}

// ------------------------------------------------- synthetic routing traces
// gen_trace (trace_gen.cpp:56-122) with TraceSpec::validate (:11-23).  One
// RNG stream per trace, consumed in the reference's order:
//   blocks : Fisher-Yates permutation of the experts (i = E-1 .. 1), then per
//            token the home block, per pick a Bernoulli(p_in) and a uniform
//            index into the eligible (untaken, in/out-of-block) experts in
//            ascending order, then the k weights;
//   uniform/zipf : per pick one uniform scaled by the remaining weight, walked
//            over untaken experts in index order; then the k weights.
// Weights: k draws from [1e-3, 1), sorted descending, divided by their sum
// (descending_weights, :44-51).
namespace {

void token_weights(occ_rng& r, int k, double* w) {
    for (int j = 0; j < k; ++j) w[j] = r.between(1e-3, 1.0);
    std::sort(w, w + k, [](double a, double b) { return a > b; });
    double sum = 0.0;
    for (int j = 0; j < k; ++j) sum += w[j];
    for (int j = 0; j < k; ++j) w[j] /= sum;
}

}  // namespace

extern "C" occ_status occ_gen_trace(const occ_trace_spec* spec, uint64_t seed, int32_t* ids, double* weights) {
    if (!spec) return occ::host_fail(OCC_ERR_ARG, "null argument");
    const int ne = spec->num_experts, k = spec->top_k, n = spec->num_tokens;
    if (ne < 1 || k < 1 || k > ne || n < 0)
        return occ::host_fail(OCC_ERR_CONFIG, "trace spec: need 1 <= top_k <= num_experts and num_tokens >= 0");
    if (spec->dist == OCC_TRACE_ZIPF && spec->alpha < 0.0)
        return occ::host_fail(OCC_ERR_CONFIG, "trace spec: zipf alpha must be >= 0");
    if (spec->dist == OCC_TRACE_BLOCKS) {
        if (spec->num_blocks < 1 || ne % spec->num_blocks != 0)
            return occ::host_fail(OCC_ERR_CONFIG, "trace spec: num_experts must be a positive multiple of num_blocks");
        if (spec->p_in < 0.0 || spec->p_in > 1.0) return occ::host_fail(OCC_ERR_CONFIG, "trace spec: p_in must be in [0, 1]");
    } else if (spec->dist != OCC_TRACE_UNIFORM && spec->dist != OCC_TRACE_ZIPF) {
        return occ::host_fail(OCC_ERR_CONFIG, "trace spec: unknown distribution");
    }
    if (n > 0 && (!ids || !weights)) return occ::host_fail(OCC_ERR_ARG, "null argument");
    occ_rng r(seed);
    std::vector<char> taken(ne);
    if (spec->dist == OCC_TRACE_BLOCKS) {
        std::vector<int> order(ne);
        std::iota(order.begin(), order.end(), 0);
        for (int i = ne - 1; i > 0; --i) std::swap(order[i], order[r.below(i + 1)]);
        const int bs = ne / spec->num_blocks;
        std::vector<int> block(ne);
        for (int pos = 0; pos < ne; ++pos) block[order[pos]] = pos / bs;
        std::vector<int> eligible;
        eligible.reserve(ne);
        for (int t = 0; t < n; ++t) {
            const int home = r.below(spec->num_blocks);
            std::fill(taken.begin(), taken.end(), 0);
            for (int j = 0; j < k; ++j) {
                const bool inside = r.unit() < spec->p_in;
                eligible.clear();
                for (int e = 0; e < ne; ++e)
                    if (!taken[e] && (block[e] == home) == inside) eligible.push_back(e);
                if (eligible.empty())  // the wanted side is exhausted: any untaken expert
                    for (int e = 0; e < ne; ++e)
                        if (!taken[e]) eligible.push_back(e);
                const int e = eligible[r.below(static_cast<int>(eligible.size()))];
                taken[e] = 1;
                ids[static_cast<size_t>(t) * k + j] = e;
            }
            token_weights(r, k, weights + static_cast<size_t>(t) * k);
        }
        return OCC_OK;
    }
    std::vector<double> mass(ne, 1.0);  // uniform == zipf with alpha 0 (same draw path)
    if (spec->dist == OCC_TRACE_ZIPF)
        for (int e = 0; e < ne; ++e) mass[e] = std::pow(static_cast<double>(e + 1), -spec->alpha);
    const double full = std::accumulate(mass.begin(), mass.end(), 0.0);
    for (int t = 0; t < n; ++t) {
        std::fill(taken.begin(), taken.end(), 0);
        double left = full;
        for (int j = 0; j < k; ++j) {
            const double target = r.unit() * left;
            double run = 0.0;
            int e_hit = -1;
            for (int e = 0; e < ne; ++e) {
                if (taken[e]) continue;
                e_hit = e;  // the last untaken expert absorbs round-off past the end
                run += mass[e];
                if (target < run) break;
            }
            taken[e_hit] = 1;
            left -= mass[e_hit];
            ids[static_cast<size_t>(t) * k + j] = e_hit;
        }
        token_weights(r, k, weights + static_cast<size_t>(t) * k);
    }
    return OCC_OK;
}

// ------------------------------------------------ component growth curve
// ComponentTracker (collab.cpp:120-169) over fixed-size token batches, from
// the per-pair first batch in which the pair co-activates (DEVICE-computed by
// occ_coactivation_first_batch): adding each batch's new edges to a
// union-find reproduces the tracker's largest component after every batch —
// components are sized over experts with at least one edge, 0 when there is
// none.
extern "C" occ_status occ_component_growth(const int32_t* first_batch, int e, int n_batches, int32_t* largest) {
    if (!first_batch || (!largest && n_batches > 0)) return occ::host_fail(OCC_ERR_ARG, "null argument");
    if (e < 1 || n_batches < 0) return occ::host_fail(OCC_ERR_SHAPE, "component_growth: bad shape");
    std::vector<std::vector<std::pair<int, int>>> new_edges(n_batches);
    for (int i = 0; i < e; ++i)
        for (int j = i + 1; j < e; ++j) {
            const int b = first_batch[static_cast<size_t>(i) * e + j];
            if (b >= 0 && b < n_batches) new_edges[b].emplace_back(i, j);
        }
    std::vector<int> parent(e), size(e, 1);
    std::iota(parent.begin(), parent.end(), 0);
    auto root = [&](int v) {
        while (parent[v] != v) v = parent[v] = parent[parent[v]];
        return v;
    };
    int best = 0;
    for (int b = 0; b < n_batches; ++b) {
        for (const auto& [i, j] : new_edges[b]) {
            int a = root(i), c = root(j);
            if (a != c) {
                if (size[a] < size[c]) std::swap(a, c);
                parent[c] = a;
                size[a] += size[c];
            }
            best = std::max(best, size[a]);
        }
        largest[b] = best;
    }
    return OCC_OK;
}
