// ref_capi.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp, never
// copied) into oracle/_ref/libmoesim_ref.so.  It exposes the reference's own
// functions through plain C signatures so that (a) the C restatement in
// oracle/occ_oracle.c is pinned against the reference itself, (b) golden
// vectors are generated from the reference (tests/golden/make_golden.py) and
// (c) bench.py's CPU baseline times the reference's own code path.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <span>
#include <thread>
#include <vector>

#include "moesim/collab.hpp"
#include "moesim/common.hpp"
#include "moesim/config.hpp"
#include "moesim/io.hpp"
#include "moesim/trace_gen.hpp"
#include "moesim/pipeline.hpp"
#include "moesim/placement.hpp"
#include "moesim/pruning.hpp"
#include "moesim/rng.hpp"
#include "moesim/routing.hpp"
#include "moesim/simnet.hpp"

using namespace moesim;

namespace {

// Same status numbering as include/occult.h (occ_status).
int status_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const ShapeError&) {
        return 1;
    } catch (const ConfigError&) {
        return 2;
    } catch (const PlacementError&) {
        return 3;
    } catch (const RoutingError&) {
        return 4;
    } catch (const CapacityError&) {
        return 5;
    } catch (const StateError&) {
        return 6;
    } catch (...) {
        return 99;
    }
}

#define GUARD(...)                              \
    try {                                       \
        __VA_ARGS__;                            \
        return 0;                               \
    } catch (...) {                             \
        return status_of(std::current_exception()); \
    }

Matrix mat(const double* p, int r, int c) {
    Matrix m(r, c);
    std::memcpy(m.data.data(), p, sizeof(double) * static_cast<size_t>(r) * c);
    return m;
}

Placement placement_of(const int* plist, int nd, int per) {
    Placement p;
    p.devices.resize(nd);
    for (int d = 0; d < nd; ++d) p.devices[d].assign(plist + d * per, plist + (d + 1) * per);
    return p;
}

RoutingOutcome routing_of(const int* ids, const double* w, int n, int k) {
    RoutingOutcome r;
    r.num_tokens = n;
    r.k = k;
    r.ids.assign(ids, ids + static_cast<size_t>(n) * k);
    r.weights.assign(w, w + static_cast<size_t>(n) * k);
    return r;
}

ExpertWeights experts_of(const double* w1, const double* w2, int ne, int dm, int dh, int act) {
    ExpertWeights ew;
    ew.num_experts = ne;
    ew.activation = static_cast<Activation>(act);
    for (int e = 0; e < ne; ++e) {
        ew.w1.push_back(mat(w1 + static_cast<size_t>(e) * dm * dh, dm, dh));
        ew.w2.push_back(mat(w2 + static_cast<size_t>(e) * dh * dm, dh, dm));
    }
    return ew;
}

}  // namespace

extern "C" {

// Reference Rng stream (rng.hpp) — used to cross-check the oracle's mt19937_64.
void ref_rng_uniform_stream(uint64_t seed, int n, double* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
}

// The CLI seed recipe (cli.cpp:248-256): master -> token, gate, expert streams.
void ref_seed_streams(uint64_t seed, uint64_t* three) {
    Rng master(seed);
    for (int i = 0; i < 3; ++i) three[i] = master.next();
}

int ref_random_matrix(uint64_t seed, int rows, int cols, int single, double* out) {
    GUARD({
        Rng r(seed);
        Matrix m = random_matrix(rows, cols, r, single ? Precision::Single : Precision::Double);
        std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
    })
}

int ref_gate_scores(const double* x, int n, int d, const double* g, int e, double* scores) {
    GUARD({
        TokenMatrix tx(mat(x, n, d), TokenState::Ori);
        GateMatrix gm{mat(g, e, d)};
        Matrix s = gate_scores(tx, gm);
        std::memcpy(scores, s.data.data(), sizeof(double) * s.data.size());
    })
}

int ref_topk_route(const double* scores, int n, int e, int k, int renorm, int* ids, double* w) {
    GUARD({
        RoutingOutcome r = topk_route(mat(scores, n, e), k, renorm != 0);
        std::memcpy(ids, r.ids.data(), sizeof(int) * r.ids.size());
        std::memcpy(w, r.weights.data(), sizeof(double) * r.weights.size());
    })
}

int ref_prune_routing(const double* scores, int n, int ne, const int* ids_in, const double* w_in, int k,
                      const int* plist, int nd, int mode, int budget, const double* sim_values,
                      int own_score, int renorm, int* ids, double* w) {
    GUARD({
        Placement p = placement_of(plist, nd, ne / nd);
        PruneSpec spec;
        spec.mode = static_cast<PruneMode>(mode);
        spec.device_budget = budget;
        spec.weight_policy = own_score ? ReplacementWeightPolicy::OwnScore : ReplacementWeightPolicy::Inherit;
        if (sim_values) {
            // Ranking exactly as the reference builds it (cli.cpp:286-300).
            SimilarityAccumulator acc(ne);
            SimilarityTable t = acc.finalize();
            t.values.assign(sim_values, sim_values + static_cast<size_t>(ne) * ne);
            t.ranking.assign(ne, {});
            for (int i = 0; i < ne; ++i) {
                for (int j = 0; j < ne; ++j)
                    if (j != i) t.ranking[i].push_back(j);
                std::stable_sort(t.ranking[i].begin(), t.ranking[i].end(), [&](int a, int b) {
                    if (t.at(i, a) != t.at(i, b)) return t.at(i, a) > t.at(i, b);
                    return a < b;
                });
            }
            spec.table = std::move(t);
        }
        RoutingOutcome out =
            prune_routing(mat(scores, n, ne), routing_of(ids_in, w_in, n, k), p, spec, renorm != 0);
        std::memcpy(ids, out.ids.data(), sizeof(int) * out.ids.size());
        std::memcpy(w, out.weights.data(), sizeof(double) * out.weights.size());
    })
}

int ref_similarity_table(const double* logits, int n, int ne, double* values, int* ranking) {
    GUARD({
        Matrix h = mat(logits, n, ne);
        SimilarityTable t = build_similarity_table({&h, 1}, ne);
        std::memcpy(values, t.values.data(), sizeof(double) * t.values.size());
        for (int i = 0; i < ne; ++i)
            std::memcpy(ranking + static_cast<size_t>(i) * (ne - 1), t.ranking[i].data(),
                        sizeof(int) * (ne - 1));
    })
}

int ref_build_dispatch_index(const int* ids, const double* w, int n, int k, const int* plist, int nd,
                             int ne, const int* tokens, int ntok, int* entries, int* n_sfd) {
    GUARD({
        DispatchIndex idx = build_dispatch_index(routing_of(ids, w, n, k), placement_of(plist, nd, ne / nd),
                                                 std::span<const int>(tokens, ntok));
        std::memcpy(entries, idx.entries.data(), sizeof(int) * idx.entries.size());
        *n_sfd = idx.n_sfd;
    })
}

int ref_accumulate_collab(const int* ids, const double* w, int n, int k, int ne, int64_t* counts) {
    GUARD({
        CollabGraph g(ne);
        for (size_t i = 0; i < g.counts.size(); ++i) g.counts[i] = counts[i];
        accumulate_collab(g, routing_of(ids, w, n, k));
        for (size_t i = 0; i < g.counts.size(); ++i) counts[i] = g.counts[i];
    })
}

int ref_normalize_graph(const int64_t* counts, int ne, double* p) {
    GUARD({
        CollabGraph g(ne);
        for (size_t i = 0; i < g.counts.size(); ++i) g.counts[i] = counts[i];
        NormGraph ng = normalize_graph(g);
        std::memcpy(p, ng.values.data(), sizeof(double) * ng.values.size());
    })
}

int ref_reschedule_placement(const double* p, int ne, int nd, int* plist) {
    GUARD({
        NormGraph g(ne);
        g.values.assign(p, p + static_cast<size_t>(ne) * ne);
        Placement out = reschedule_placement(g, nd);
        for (int d = 0; d < nd; ++d)
            std::memcpy(plist + static_cast<size_t>(d) * (ne / nd), out.devices[d].data(),
                        sizeof(int) * (ne / nd));
    })
}

// forward_given_routing (pipeline.cpp:360-501) with its saved index state.
// Output layout identical to orc_forward_given_routing.
struct ref_report {
    double mean_replicas, cap_replicas, intra_share, inter_share;
    long long cross_device_bytes;
    long long crossing_rows;
    long long per_device_rows[64];
    int n_sfd_src[64];
    int n_epd_dev[64];
};

int ref_forward_given_routing(const double* x, int n, int dm, const int* ids, const double* w, int k,
                              const double* w1, const double* w2, int ne, int dh, const int* plist, int nd,
                              const int* sources, int act, int single, int bytes_per_scalar,
                              double cap_replicas, double* x_out, ref_report* rep, int* dindex_out,
                              int* inbox_token, int* inbox_source, int* inbox_slot, int* cindex_out) {
    GUARD({
        MoEConfig cfg;
        cfg.num_experts = ne;
        cfg.top_k = k;
        cfg.num_devices = nd;
        cfg.embed_dim = dm;
        cfg.hidden_dim = dh;
        cfg.precision = single ? Precision::Single : Precision::Double;
        cfg.activation = static_cast<Activation>(act);
        TokenMatrix tx(mat(x, n, dm), TokenState::Ori);
        ForwardState st;
        ForwardResult res = forward_given_routing(
            tx, routing_of(ids, w, n, k), experts_of(w1, w2, ne, dm, dh, act), placement_of(plist, nd, ne / nd),
            cfg, std::span<const int>(sources, n), bytes_per_scalar, cap_replicas, &st);
        std::memcpy(x_out, res.x_out.values.data.data(), sizeof(double) * res.x_out.values.data.size());
        if (rep) {
            rep->mean_replicas = res.report.mean_replicas;
            rep->cap_replicas = res.report.cap_replicas;
            rep->intra_share = res.report.intra_share;
            rep->inter_share = res.report.inter_share;
            rep->cross_device_bytes = res.report.cross_device_bytes;
            rep->crossing_rows = bytes_per_scalar ? res.report.cross_device_bytes / (static_cast<long long>(dm) * bytes_per_scalar) : 0;
            for (int d = 0; d < nd; ++d) rep->per_device_rows[d] = res.report.per_device_token_counts[d];
            for (int s = 0; s < nd; ++s) rep->n_sfd_src[s] = st.dindex[s].n_sfd;
            for (int d = 0; d < nd; ++d) rep->n_epd_dev[d] = st.shards[d].cindex.n_epd;
        }
        size_t dpos = 0, ipos = 0, cpos = 0;
        for (int s = 0; s < nd; ++s) {
            if (dindex_out) std::memcpy(dindex_out + dpos, st.dindex[s].entries.data(), sizeof(int) * st.dindex[s].entries.size());
            dpos += st.dindex[s].entries.size();
        }
        for (int d = 0; d < nd; ++d) {
            const ShardRecord& sh = st.shards[d];
            if (inbox_token) {
                std::memcpy(inbox_token + ipos, sh.row_token.data(), sizeof(int) * sh.row_token.size());
                std::memcpy(inbox_source + ipos, sh.row_source.data(), sizeof(int) * sh.row_source.size());
                std::memcpy(inbox_slot + ipos, sh.row_source_slot.data(), sizeof(int) * sh.row_source_slot.size());
            }
            ipos += sh.row_token.size();
            if (cindex_out) std::memcpy(cindex_out + cpos, sh.cindex.entries.data(), sizeof(int) * sh.cindex.entries.size());
            cpos += sh.cindex.entries.size();
        }
    })
}

// backward_vjps (backward.cpp:24-161) after a saving forward_given_routing.
// Outputs: gx [n, dm], gw1 [ne, dm, dh], gw2 [ne, dh, dm], gr [n, k].
int ref_backward(const double* x, int n, int dm, const int* ids, const double* w, int k, const double* w1,
                 const double* w2, int ne, int dh, const int* plist, int nd, const int* sources, int act, int single,
                 const double* upstream, double* gx, double* gw1, double* gw2, double* gr) {
    GUARD({
        MoEConfig cfg;
        cfg.num_experts = ne;
        cfg.top_k = k;
        cfg.num_devices = nd;
        cfg.embed_dim = dm;
        cfg.hidden_dim = dh;
        cfg.precision = single ? Precision::Single : Precision::Double;
        cfg.activation = static_cast<Activation>(act);
        TokenMatrix tx(mat(x, n, dm), TokenState::Ori);
        ForwardState st;
        (void)forward_given_routing(tx, routing_of(ids, w, n, k), experts_of(w1, w2, ne, dm, dh, act),
                                    placement_of(plist, nd, ne / nd), cfg, std::span<const int>(sources, n), 4, -1.0,
                                    &st);
        Gradients g = backward_vjps(mat(upstream, n, dm), st);
        std::memcpy(gx, g.x.data.data(), sizeof(double) * g.x.data.size());
        for (int e = 0; e < ne; ++e) {
            std::memcpy(gw1 + static_cast<size_t>(e) * dm * dh, g.w1[e].data.data(), sizeof(double) * dm * dh);
            std::memcpy(gw2 + static_cast<size_t>(e) * dh * dm, g.w2[e].data.data(), sizeof(double) * dh * dm);
        }
        std::memcpy(gr, g.routing_weights.data(), sizeof(double) * g.routing_weights.size());
    })
}

int ref_dense_given_routing(const double* x, int n, int dm, const int* ids, const double* w, int k,
                            const double* w1, const double* w2, int ne, int dh, int act, int single,
                            double* out) {
    GUARD({
        TokenMatrix tx(mat(x, n, dm), TokenState::Ori);
        TokenMatrix o = dense_given_routing(tx, routing_of(ids, w, n, k), experts_of(w1, w2, ne, dm, dh, act),
                                            single ? Precision::Single : Precision::Double);
        std::memcpy(out, o.values.data.data(), sizeof(double) * o.values.data.size());
    })
}

// CPU baseline: gate_scores + topk_route + forward_given_routing, the
// reference's own path (cli.cpp:271-316), on `nthreads` independent token
// chunks in parallel (the reference functions are pure).
// Returns the number of tokens processed.
// A reference "layer session": the experts, gate, placement and config are
// converted to the reference's own types once (as a caller of the moesim
// library would hold them); ref_session_forward then times only the
// reference's forward_expert_parallel (pipeline.cpp:503-517) on `nthreads`
// token shards.
struct RefSession {
    ExpertWeights ew;
    GateMatrix gm;
    Placement pl;
    MoEConfig cfg;
};

void* ref_session_create(const double* gate, int ne, int k, const double* w1, const double* w2, int dm, int dh,
                         int nd, int act, int single) {
    try {
        auto* s = new RefSession{experts_of(w1, w2, ne, dm, dh, act), GateMatrix{mat(gate, ne, dm)},
                                 trivial_placement(ne, nd), MoEConfig{}};
        s->cfg.num_experts = ne;
        s->cfg.top_k = k;
        s->cfg.num_devices = nd;
        s->cfg.embed_dim = dm;
        s->cfg.hidden_dim = dh;
        s->cfg.precision = single ? Precision::Single : Precision::Double;
        s->cfg.activation = static_cast<Activation>(act);
        return s;
    } catch (...) {
        return nullptr;
    }
}

void ref_session_destroy(void* s) { delete static_cast<RefSession*>(s); }

int ref_session_forward(void* sp, const double* x, int n, int nthreads, double* x_out) {
    RefSession& s = *static_cast<RefSession*>(sp);
    const int dm = s.cfg.embed_dim;
    std::vector<std::thread> pool;
    std::vector<int> rc(nthreads, 0);
    const int chunk = (n + nthreads - 1) / nthreads;
    for (int th = 0; th < nthreads; ++th) {
        pool.emplace_back([&, th] {
            const int lo = th * chunk, hi = std::min(n, lo + chunk);
            if (lo >= hi) return;
            try {
                TokenMatrix tx(mat(x + static_cast<size_t>(lo) * dm, hi - lo, dm), TokenState::Ori);
                ForwardResult res = forward_expert_parallel(tx, s.gm, s.ew, s.pl, PruneSpec{}, s.cfg);
                std::memcpy(x_out + static_cast<size_t>(lo) * dm, res.x_out.values.data.data(),
                            sizeof(double) * res.x_out.values.data.size());
            } catch (...) {
                rc[th] = status_of(std::current_exception());
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int v : rc)
        if (v) return -v;
    return n;
}

int ref_forward_expert_parallel_mt(const double* x, int n, int dm, const double* gate, int ne, int k,
                                   const double* w1, const double* w2, int dh, int nd, int act, int single,
                                   int nthreads, double* x_out) {
    std::vector<std::thread> pool;
    std::vector<int> rc(nthreads, 0);
    ExpertWeights ew = experts_of(w1, w2, ne, dm, dh, act);
    GateMatrix gm{mat(gate, ne, dm)};
    Placement pl = trivial_placement(ne, nd);
    MoEConfig cfg;
    cfg.num_experts = ne;
    cfg.top_k = k;
    cfg.num_devices = nd;
    cfg.embed_dim = dm;
    cfg.hidden_dim = dh;
    cfg.precision = single ? Precision::Single : Precision::Double;
    cfg.activation = static_cast<Activation>(act);
    const int chunk = (n + nthreads - 1) / nthreads;
    for (int th = 0; th < nthreads; ++th) {
        pool.emplace_back([&, th] {
            const int lo = th * chunk, hi = std::min(n, lo + chunk);
            if (lo >= hi) return;
            try {
                TokenMatrix tx(mat(x + static_cast<size_t>(lo) * dm, hi - lo, dm), TokenState::Ori);
                ForwardResult res = forward_expert_parallel(tx, gm, ew, pl, PruneSpec{}, cfg);
                std::memcpy(x_out + static_cast<size_t>(lo) * dm, res.x_out.values.data.data(),
                            sizeof(double) * res.x_out.values.data.size());
            } catch (...) {
                rc[th] = status_of(std::current_exception());
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int v : rc)
        if (v) return -v;
    return n;
}

}  // extern "C"

// ---------------------------------------------------- formats (io.cpp) ----
// Text results go to (buf, cap); the return value is the full length (the
// caller retries with a larger buffer when it exceeds cap), or -1 with the
// exception text in buf.
namespace {
long long emit(const std::string& text, char* buf, long long cap) {
    if (buf && cap > 0) {
        const size_t m = std::min<size_t>(text.size(), static_cast<size_t>(cap - 1));
        std::memcpy(buf, text.data(), m);
        buf[m] = 0;
    }
    return static_cast<long long>(text.size());
}
}  // namespace

extern "C" {

long long ref_gen_trace_text(int dist, int ne, int k, int n, double alpha, int blocks, double p_in, const char* tag,
                             uint64_t seed, char* buf, long long cap) {
    try {
        TraceSpec spec;
        spec.dist = static_cast<TraceSpec::Dist>(dist);
        spec.num_experts = ne;
        spec.top_k = k;
        spec.num_tokens = n;
        spec.alpha = alpha;
        spec.num_blocks = blocks;
        spec.p_in = p_in;
        spec.tag = tag ? tag : "";
        std::ostringstream os;
        write_trace(os, gen_trace(spec, seed));
        return emit(os.str(), buf, cap);
    } catch (const std::exception& e) {
        emit(e.what(), buf, cap);
        return -1;
    }
}

// read_* then write_* of the parsed value (the round trip), or the error.
long long ref_roundtrip_text(int kind, const char* text, char* buf, long long cap) {
    try {
        std::istringstream is(text);
        std::ostringstream os;
        if (kind == 0) write_trace(os, read_trace(is));
        else if (kind == 1) write_matrix(os, read_matrix(is));
        else write_placement(os, read_placement(is));
        return emit(os.str(), buf, cap);
    } catch (const std::exception& e) {
        emit(e.what(), buf, cap);
        return -1;
    }
}

long long ref_write_matrix_text(const double* m, int rows, int cols, char* buf, long long cap) {
    std::ostringstream os;
    write_matrix(os, mat(m, rows, cols));
    return emit(os.str(), buf, cap);
}

long long ref_write_placement_text(const int* plist, int nd, int per, char* buf, long long cap) {
    std::ostringstream os;
    write_placement(os, placement_of(plist, nd, per));
    return emit(os.str(), buf, cap);
}

// ComponentTracker over `batch`-token slices (cli.cpp:131-145): points as
// (tokens_seen, largest); returns the point count.
int ref_component_points(const int* ids, int n, int k, int ne, int batch, long long* tokens, int* largest) {
    ComponentTracker tr(ne);
    std::vector<double> w(static_cast<size_t>(n) * k, 1.0 / k);
    for (int t0 = 0; t0 < n; t0 += batch) {
        const int t1 = std::min(n, t0 + batch);
        tr.add(routing_of(ids + static_cast<size_t>(t0) * k, w.data() + static_cast<size_t>(t0) * k, t1 - t0, k));
    }
    const auto& pts = tr.points();
    for (size_t i = 0; i < pts.size(); ++i) {
        tokens[i] = pts[i].first;
        largest[i] = pts[i].second;
    }
    return static_cast<int>(pts.size());
}

}  // extern "C"

extern "C" {


}  // extern "C"
