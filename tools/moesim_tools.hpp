// moesim_tools.hpp — host-side helpers of the moesim_gpu command line that are
// NOT part of the B200 layer (test-input generation and trace statistics,
// SURVEY §2 rows 4 and 10): the reference's RNG streams (rng.hpp:12-38),
// gen_trace (trace_gen.cpp:11-122) and ComponentTracker (collab.cpp:120-169).
// Kept out of libocc so the product ABI exports only the layer, profiling and
// placement API.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <string>
#include <utility>
#include <vector>

namespace tools {

enum TraceDist { kUniform = 0, kZipf = 1, kBlocks = 2 };
struct TraceSpec {  // trace_gen.hpp:12-33
    int dist;
    int num_experts;
    int top_k;
    int num_tokens;
    double alpha;
    int num_blocks;
    double p_in;
};

// ------------------------------------------------------- deterministic RNG
// rng.hpp:12-38: std::mt19937_64 (its output sequence is fixed by the C++
// standard) with the reference's own derived draws, so streams, synthetic
// inputs and traces are identical to the reference CLI's for the same seed.
struct Rng {
    std::mt19937_64 g;
    explicit Rng(uint64_t seed) : g(seed) {}
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


// random_matrix (core.cpp:54-58): row-major uniform [-1, 1), rounded through
// float for single precision.
inline void rng_matrix(Rng* r, int rows, int cols, int single, double* out) {
    const size_t n = static_cast<size_t>(rows) * cols;
    for (size_t i = 0; i < n; ++i) {
        const double v = r->between(-1.0, 1.0);
        out[i] = single ? static_cast<double>(static_cast<float>(v)) : v;
    }
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
inline void token_weights(Rng& r, int k, double* w) {
    for (int j = 0; j < k; ++j) w[j] = r.between(1e-3, 1.0);
    std::sort(w, w + k, [](double a, double b) { return a > b; });
    double sum = 0.0;
    for (int j = 0; j < k; ++j) sum += w[j];
    for (int j = 0; j < k; ++j) w[j] /= sum;
}

// Returns "" or TraceSpec::validate's message.
inline std::string gen_trace(const TraceSpec* spec, uint64_t seed, int32_t* ids, double* weights) {
    const int ne = spec->num_experts, k = spec->top_k, n = spec->num_tokens;
    if (ne < 1 || k < 1 || k > ne || n < 0)
        return "trace spec: need 1 <= top_k <= num_experts and num_tokens >= 0";
    if (spec->dist == kZipf && spec->alpha < 0.0)
        return "trace spec: zipf alpha must be >= 0";
    if (spec->dist == kBlocks) {
        if (spec->num_blocks < 1 || ne % spec->num_blocks != 0)
            return "trace spec: num_experts must be a positive multiple of num_blocks";
        if (spec->p_in < 0.0 || spec->p_in > 1.0) return "trace spec: p_in must be in [0, 1]";
    } else if (spec->dist != kUniform && spec->dist != kZipf) {
        return "trace spec: unknown distribution";
    }
    Rng r(seed);
    std::vector<char> taken(ne);
    if (spec->dist == kBlocks) {
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
        return "";
    }
    std::vector<double> mass(ne, 1.0);  // uniform == zipf with alpha 0 (same draw path)
    if (spec->dist == kZipf)
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
    return "";
}

// ------------------------------------------------ component growth curve
// ComponentTracker (collab.cpp:120-169) over fixed-size token batches, from
// the per-pair first batch in which the pair co-activates (first_batch_of below): adding each batch's new edges to a
// union-find reproduces the tracker's largest component after every batch —
// components are sized over experts with at least one edge, 0 when there is
// none.
inline void component_growth(const int32_t* first_batch, int e, int n_batches, int32_t* largest) {
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
}

// Per expert pair (i < j): the first batch (t / batch) in which both are
// routed together, INT32_MAX when never -- the edges ComponentTracker adds.
inline std::vector<int32_t> first_batch_of(const int32_t* ids, int n, int k, int e, int batch) {
    std::vector<int32_t> first(static_cast<size_t>(e) * e, INT32_MAX);
    for (int t = 0; t < n; ++t)
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) {
                const int i = ids[static_cast<size_t>(t) * k + a], j = ids[static_cast<size_t>(t) * k + b];
                if (i < j) first[static_cast<size_t>(i) * e + j] = std::min(first[static_cast<size_t>(i) * e + j], t / batch);
            }
    return first;
}

}  // namespace tools
