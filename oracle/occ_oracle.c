/*
 * occ_oracle.c — CPU restatement of the reference ("moesim") hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path; it is never linked into, loaded by, or called from
 * the product (`paper_2505_13345_b200/`).  Only `tests/`,
 * `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
 * reference` legs may load it.
 *
 * Parity pinning: every function below is checked against the reference
 * itself (oracle/_ref/libmoesim_ref.so, compiled from
 * /root/reference/proj/src by oracle/Makefile) and against the golden
 * vectors under tests/golden/ (tests/test_oracle.py).
 *
 * Numerics follow the reference exactly: values are doubles, dot products
 * accumulate in double in ascending-k order with no FMA contraction
 * (build with -ffp-contract=off), Precision::Single rounds through float at
 * every op boundary (reference common.hpp:38-42).
 *
 * Citations are to /root/reference/proj/<file>:<line>.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE 1
#define ORC_CONFIG 2
#define ORC_PLACEMENT 3
#define ORC_ROUTING 4
#define ORC_CAPACITY 5

/* ---------------------------------------------------------------- rng --- */
/* std::mt19937_64 (fully specified by the C++ standard) + the reference's
 * distribution-free draws (include/moesim/rng.hpp:14-38). */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static void orc_rng_twist(orc_rng* r) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
        uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->idx >= 312) orc_rng_twist(r);
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:21 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:23 */
double orc_rng_uniform_range(orc_rng* r, double lo, double hi) {
    return lo + (hi - lo) * orc_rng_uniform(r);
}
/* rng.hpp:26-34 */
int orc_rng_uniform_int(orc_rng* r, int n) {
    const uint64_t un = (uint64_t)n;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % un;
    uint64_t v;
    do { v = orc_rng_next(r); } while (v >= limit);
    return (int)(v % un);
}

size_t orc_rng_size(void) { return sizeof(orc_rng); }

static inline double quant(double v, int single) { return single ? (double)(float)v : v; }

/* core.cpp:54-58: uniform [-1,1) rounded to the storage precision. */
void orc_random_matrix(orc_rng* r, int rows, int cols, int single, double* out) {
    for (long i = 0; i < (long)rows * cols; ++i) out[i] = quant(orc_rng_uniform_range(r, -1.0, 1.0), single);
}

/* ------------------------------------------------------------ routing --- */
/* routing.cpp:33-52: logits = x * g^T (double, ascending k), softmax with
 * per-row max subtraction. */
void orc_gate_logits(const double* x, int n, int d, const double* g, int e, double* logits) {
    for (int t = 0; t < n; ++t)
        for (int j = 0; j < e; ++j) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += x[(long)t * d + c] * g[(long)j * d + c];
            logits[(long)t * e + j] = acc;
        }
}

void orc_softmax_rows(double* s, int n, int e) {
    for (int t = 0; t < n; ++t) {
        double* row = s + (long)t * e;
        double mx = row[0];
        for (int j = 1; j < e; ++j)
            if (row[j] > mx) mx = row[j];
        double sum = 0.0;
        for (int j = 0; j < e; ++j) {
            row[j] = exp(row[j] - mx);
            sum += row[j];
        }
        for (int j = 0; j < e; ++j) row[j] /= sum;
    }
}

void orc_gate_scores(const double* x, int n, int d, const double* g, int e, double* scores) {
    orc_gate_logits(x, n, d, g, e, scores);
    orc_softmax_rows(scores, n, e);
}

/* (score desc, index asc) — routing.cpp:71-74 */
static inline int orc_before(const double* row, int a, int b) {
    if (row[a] != row[b]) return row[a] > row[b];
    return a < b;
}

/* routing.cpp:54-58 */
static int orc_renorm(double* w, int k) {
    double sum = 0.0;
    for (int j = 0; j < k; ++j) sum += w[j];
    if (sum <= 0.0) return ORC_ROUTING;
    for (int j = 0; j < k; ++j) w[j] /= sum;
    return ORC_OK;
}

/* Full order of one score row under (score desc, index asc). */
static void orc_order(const double* row, int e, int* order) {
    for (int j = 0; j < e; ++j) order[j] = j;
    for (int i = 1; i < e; ++i) { /* insertion sort: stable, total order */
        int v = order[i], p = i - 1;
        while (p >= 0 && orc_before(row, v, order[p])) { order[p + 1] = order[p]; --p; }
        order[p + 1] = v;
    }
}

/* routing.cpp:60-84 */
int orc_topk_route(const double* scores, int n, int e, int k, int renormalize, int* ids, double* w) {
    if (k < 1 || k > e) return ORC_ROUTING;
    int* order = (int*)malloc(sizeof(int) * (size_t)e);
    for (int t = 0; t < n; ++t) {
        const double* row = scores + (long)t * e;
        orc_order(row, e, order);
        for (int j = 0; j < k; ++j) {
            ids[(long)t * k + j] = order[j];
            w[(long)t * k + j] = row[order[j]];
        }
        if (renormalize && orc_renorm(w + (long)t * k, k)) { free(order); return ORC_ROUTING; }
    }
    free(order);
    return ORC_OK;
}

/* ---------------------------------------------------------- placement --- */
/* placement.cpp:17-30; returns ORC_PLACEMENT if not a partition. */
int orc_expert_to_device(const int* plist, int nd, int per, int* dev_of) {
    const int n = nd * per;
    for (int i = 0; i < n; ++i) dev_of[i] = -1;
    for (int d = 0; d < nd; ++d)
        for (int i = 0; i < per; ++i) {
            int e = plist[d * per + i];
            if (e < 0 || e >= n || dev_of[e] >= 0) return ORC_PLACEMENT;
            dev_of[e] = d;
        }
    return ORC_OK;
}

/* placement.cpp:47-58 */
void orc_trivial_placement(int ne, int nd, int* plist) {
    const int per = ne / nd;
    for (int d = 0; d < nd; ++d)
        for (int i = 0; i < per; ++i) plist[d * per + i] = d * per + i;
}

/* placement.cpp:80-84: mean in member-list order. */
static double orc_mean_against(const double* p, int ne, const int* members, int m, int e) {
    double sum = 0.0;
    for (int i = 0; i < m; ++i) sum += p[(long)members[i] * ne + e];
    return sum / (double)m;
}

/* placement.cpp:88-148 (Alg. 1). plist: nd x per, list order significant. */
int orc_reschedule_placement(const double* p, int ne, int nd, int* plist) {
    if (nd < 1 || ne < 1 || ne % nd) return ORC_CONFIG;
    const int per = ne / nd;
    char* used = (char*)calloc((size_t)ne, 1);
    int* used_list = (int*)malloc(sizeof(int) * (size_t)ne);
    int n_used = 0;
    for (int d = 0; d < nd; ++d) {
        int* local = plist + d * per;
        int n_local = 0;
#define TAKE(e_) do { local[n_local++] = (e_); used[(e_)] = 1; used_list[n_used++] = (e_); } while (0)
        if (d == 0) {
            if (ne == 1) {
                TAKE(0);
            } else {
                int bi = 0, bj = 1; /* placement.cpp:63-76 */
                double best = -1.0;
                for (int i = 0; i < ne; ++i)
                    for (int j = i + 1; j < ne; ++j)
                        if (p[(long)i * ne + j] > best) { best = p[(long)i * ne + j]; bi = i; bj = j; }
                TAKE(bi);
                if (per >= 2) TAKE(bj);
            }
        } else {
            int pick = -1;
            double best = 0.0;
            for (int e = 0; e < ne; ++e) {
                if (used[e]) continue;
                double s = orc_mean_against(p, ne, used_list, n_used, e);
                if (pick < 0 || s < best) { best = s; pick = e; }
            }
            TAKE(pick);
        }
        while (n_local < per) {
            int pick = -1;
            double best = 0.0;
            for (int e = 0; e < ne; ++e) {
                if (used[e]) continue;
                double s = orc_mean_against(p, ne, local, n_local, e);
                if (pick < 0 || s > best) { best = s; pick = e; }
            }
            TAKE(pick);
        }
#undef TAKE
    }
    free(used);
    free(used_list);
    return ORC_OK;
}

/* ------------------------------------------------------------- collab --- */
/* collab.cpp:10-23: counts is ne x ne int64, accumulated in place. */
int orc_accumulate_collab(const int* ids, int n, int k, int ne, int64_t* counts) {
    for (int t = 0; t < n; ++t) {
        const int* row = ids + (long)t * k;
        for (int a = 0; a < k; ++a) {
            if (row[a] < 0 || row[a] >= ne) return ORC_ROUTING;
            for (int b = a + 1; b < k; ++b) {
                counts[(long)row[a] * ne + row[b]] += 1;
                counts[(long)row[b] * ne + row[a]] += 1;
            }
        }
    }
    return ORC_OK;
}

/* collab.cpp:31-39 */
void orc_normalize_graph(const int64_t* counts, int ne, double* p) {
    int64_t mx = 0;
    for (long i = 0; i < (long)ne * ne; ++i)
        if (counts[i] > mx) mx = counts[i];
    for (long i = 0; i < (long)ne * ne; ++i) p[i] = mx == 0 ? 0.0 : (double)counts[i] / (double)mx;
}

/* collab.cpp:41-61 */
double orc_mean_token_replicas(const int* ids, int n, int k, const int* dev_of, int nd) {
    if (n == 0) return 0.0;
    long long total = 0;
    char* seen = (char*)malloc((size_t)nd);
    for (int t = 0; t < n; ++t) {
        memset(seen, 0, (size_t)nd);
        for (int j = 0; j < k; ++j) {
            int d = dev_of[ids[(long)t * k + j]];
            if (!seen[d]) { seen[d] = 1; ++total; }
        }
    }
    free(seen);
    return (double)total / n;
}

/* collab.cpp:105-118 */
void orc_collaboration_shares(const int* ids, int n, int k, const int* dev_of, double* intra,
                              double* inter) {
    long long a_in = 0, a_out = 0;
    for (int t = 0; t < n; ++t) {
        const int* row = ids + (long)t * k;
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) {
                if (dev_of[row[a]] == dev_of[row[b]]) ++a_in; else ++a_out;
            }
    }
    long long tot = a_in + a_out;
    *intra = tot ? (double)a_in / tot : 0.0;
    *inter = tot ? (double)a_out / tot : 0.0;
}

/* ------------------------------------------------------------ pruning --- */
/* pruning.cpp:21-33. Returns the number of allowed devices. */
static int orc_allowed_devices(const int* ids, int k, const int* dev_of, int budget, int* devs) {
    int n = 0;
    for (int j = 0; j < k; ++j) {
        int d = dev_of[ids[j]], found = 0;
        for (int i = 0; i < n; ++i) found |= devs[i] == d;
        if (!found) {
            if (n == budget) break;
            devs[n++] = d;
        }
    }
    return n;
}

/* pruning.cpp:35-64 */
int orc_prune_router_score(const double* row, int ne, const int* dev_of, int nd, int budget, int k,
                           int renormalize, int* ids, double* w) {
    int* order = (int*)malloc(sizeof(int) * (size_t)ne);
    int* devs = (int*)malloc(sizeof(int) * (size_t)nd);
    char* in_range = (char*)calloc((size_t)nd, 1);
    orc_order(row, ne, order);
    int na = orc_allowed_devices(order, k, dev_of, budget, devs);
    for (int i = 0; i < na; ++i) in_range[devs[i]] = 1;
    int m = 0;
    for (int i = 0; i < ne && m < k; ++i) {
        int e = order[i];
        if (!in_range[dev_of[e]]) continue;
        ids[m] = e;
        w[m] = row[e];
        ++m;
    }
    free(order); free(devs); free(in_range);
    if (m < k) return ORC_CAPACITY;
    if (renormalize) return orc_renorm(w, k);
    return ORC_OK;
}

/* pruning.cpp:66-122. ranking: ne x (ne-1), per expert most-similar first. */
int orc_prune_similarity(const int* ids_in, const double* row, int ne, const int* dev_of, int nd,
                         int budget, int k, const int* ranking, int own_score, int renormalize,
                         int* ids, double* w) {
    int* devs = (int*)malloc(sizeof(int) * (size_t)nd);
    char* in_range = (char*)calloc((size_t)nd, 1);
    char* selected = (char*)calloc((size_t)ne, 1);
    char* replaced = (char*)calloc((size_t)k, 1);
    int rc = ORC_OK;
    int na = orc_allowed_devices(ids_in, k, dev_of, budget, devs);
    for (int i = 0; i < na; ++i) in_range[devs[i]] = 1;
    for (int j = 0; j < k; ++j)
        if (in_range[dev_of[ids_in[j]]]) selected[ids_in[j]] = 1;
    for (int j = 0; j < k; ++j) {
        int e = ids_in[j];
        if (in_range[dev_of[e]]) { ids[j] = e; continue; }
        int pick = -1;
        for (int c = 0; c < ne - 1; ++c) {
            int cand = ranking[(long)e * (ne - 1) + c];
            if (!in_range[dev_of[cand]] || selected[cand]) continue;
            pick = cand;
            break;
        }
        if (pick < 0) { rc = ORC_CAPACITY; goto done; }
        selected[pick] = 1;
        ids[j] = pick;
        replaced[j] = 1;
    }
    /* pruned_weight_policy, pruning.cpp:124-139; original = raw scores */
    for (int j = 0; j < k; ++j) w[j] = (own_score && replaced[j]) ? row[ids[j]] : row[ids_in[j]];
    if (renormalize && (rc = orc_renorm(w, k))) goto done;
    if (own_score) { /* pruning.cpp:106-119: re-sort by (weight desc, id asc) */
        for (int i = 1; i < k; ++i) {
            int vi = ids[i];
            double vw = w[i];
            int p = i - 1;
            while (p >= 0 && (vw > w[p] || (vw == w[p] && vi < ids[p]))) {
                ids[p + 1] = ids[p]; w[p + 1] = w[p]; --p;
            }
            ids[p + 1] = vi; w[p + 1] = vw;
        }
    }
done:
    free(devs); free(in_range); free(selected); free(replaced);
    return rc;
}

/* pruning.cpp:141-163. mode: 0 none, 1 router score, 2 similarity. */
int orc_prune_routing(const double* scores, int n, int ne, const int* ids_in, const double* w_in, int k,
                      const int* dev_of, int nd, int mode, int budget, const int* ranking,
                      int own_score, int renormalize, int* ids, double* w) {
    if (mode == 0) {
        memcpy(ids, ids_in, sizeof(int) * (size_t)n * k);
        memcpy(w, w_in, sizeof(double) * (size_t)n * k);
        return ORC_OK;
    }
    if (budget < 1 || budget > nd) return ORC_CONFIG;
    if (mode == 2 && !ranking) return ORC_CONFIG;
    for (int t = 0; t < n; ++t) {
        int rc = mode == 1
                     ? orc_prune_router_score(scores + (long)t * ne, ne, dev_of, nd, budget, k,
                                              renormalize, ids + (long)t * k, w + (long)t * k)
                     : orc_prune_similarity(ids_in + (long)t * k, scores + (long)t * ne, ne, dev_of,
                                            nd, budget, k, ranking, own_score, renormalize,
                                            ids + (long)t * k, w + (long)t * k);
        if (rc) return rc;
    }
    return ORC_OK;
}

/* pruning.cpp:170-219: squared-cosine table + rankings from logits. */
void orc_similarity_table(const double* logits, int n, int ne, double* values, int* ranking) {
    double* inner = (double*)calloc((size_t)ne * ne, sizeof(double));
    for (int i = 0; i < ne; ++i)
        for (int j = i; j < ne; ++j) {
            double dot = 0.0;
            for (int t = 0; t < n; ++t) dot += logits[(long)t * ne + i] * logits[(long)t * ne + j];
            inner[(long)i * ne + j] += dot;
            if (i != j) inner[(long)j * ne + i] += dot;
        }
    const double nn = n > 0 ? (double)n : 1.0;
    for (int i = 0; i < ne; ++i)
        for (int j = 0; j < ne; ++j) {
            double si = inner[(long)i * ne + i], sj = inner[(long)j * ne + j];
            double v = 0.0;
            if (!(si <= 0.0 || sj <= 0.0)) {
                double mean_ip = inner[(long)i * ne + j] / nn;
                double denom = (si / nn) * (sj / nn);
                v = mean_ip * mean_ip / denom;
                if (v > 1.0) v = 1.0;
            }
            values[(long)i * ne + j] = v;
        }
    for (int i = 0; i < ne; ++i) {
        int* rk = ranking + (long)i * (ne - 1);
        int m = 0;
        for (int j = 0; j < ne; ++j)
            if (j != i) rk[m++] = j;
        const double* row = values + (long)i * ne;
        for (int a = 1; a < m; ++a) { /* stable insertion sort */
            int v = rk[a], p = a - 1;
            while (p >= 0 && (row[v] > row[rk[p]] || (row[v] == row[rk[p]] && v < rk[p]))) {
                rk[p + 1] = rk[p]; --p;
            }
            rk[p + 1] = v;
        }
    }
    free(inner);
}

/* ---------------------------------------------------------- EP path ---- */
/* pipeline.cpp:24-50 (BRIM0). tokens: the source's ascending Ori rows.
 * entries: nd x ntok. Returns n_sfd. */
int orc_build_dispatch_index(const int* ids, int k, const int* dev_of, int nd, const int* tokens,
                             int ntok, int* entries) {
    int ctr = 0;
    for (int d = 0; d < nd; ++d)
        for (int i = 0; i < ntok; ++i) {
            int hit = 0;
            for (int j = 0; j < k; ++j)
                if (dev_of[ids[(long)tokens[i] * k + j]] == d) { hit = 1; break; }
            entries[(long)d * ntok + i] = hit ? ctr++ : -1;
        }
    return ctr;
}

/* pipeline.cpp:52-89 (BRIM1). member: n_loc x rows 0/1 flags (already
 * validated).  entries: n_loc x rows. Returns n_epd. */
static int orc_compute_index_from_member(const char* member, int n_loc, int rows, int* entries) {
    int ctr = 0;
    for (int e = 0; e < n_loc; ++e)
        for (int t = 0; t < rows; ++t)
            entries[(long)e * rows + t] = member[(long)e * rows + t] ? ctr++ : -1;
    return ctr;
}

static double act_fn(double v, int act) {
    if (act == 2) return v > 0.0 ? v : 0.0;            /* ReLU */
    if (act == 1) return v / (1.0 + exp(-v));          /* SiLU */
    return v;                                          /* Identity */
}

/* Result record of orc_forward_given_routing (reference ForwardResult +
 * the saved index state of ForwardState, pipeline.hpp:133-165). */
typedef struct {
    double mean_replicas, cap_replicas, intra_share, inter_share;
    long long cross_device_bytes;
    long long crossing_rows;
    long long per_device_rows[64]; /* Sfd rows received per device */
    int n_sfd_src[64];             /* per source */
    int n_epd_dev[64];             /* per device */
} orc_report;

/*
 * pipeline.cpp:360-501 forward_given_routing, restated.
 *   x: n x dm (Ori), ids/w: n x k, w1: ne x dm x dh, w2: ne x dh x dm,
 *   w3 (optional, NULL = reference 2-matrix expert): ne x dm x dh, gated
 *   SwiGLU extension h = silu(x w1) * (x w3) — NOT in the reference
 *   (SPEC.md:73), parity of that mode is pinned against torch fp64.
 *   plist: nd x per placement lists (order significant), sources: n ints.
 * Optional outputs (may be NULL):
 *   dindex_out: concat over sources s of nd x ntok_s BRIM0 matrices
 *   inbox_token/source/slot: concat over devices of per-inbox-row records
 *   cindex_out: concat over devices of per x rows_d BRIM1 matrices
 */
int orc_forward_given_routing(const double* x, int n, int dm, const int* ids, const double* w, int k,
                              const double* w1, const double* w2, const double* w3, int ne, int dh,
                              const int* plist, int nd, const int* sources, int act, int single,
                              int bytes_per_scalar, double cap_replicas, double* x_out,
                              orc_report* rep, int* dindex_out, int* inbox_token, int* inbox_source,
                              int* inbox_slot, int* cindex_out) {
    if (nd < 1 || nd > 64 || ne < 1 || ne % nd) return ORC_CONFIG;
    const int per = ne / nd;
    int* dev_of = (int*)malloc(sizeof(int) * (size_t)ne);
    if (orc_expert_to_device(plist, nd, per, dev_of)) { free(dev_of); return ORC_PLACEMENT; }
    for (long i = 0; i < (long)n * k; ++i)
        if (ids[i] < 0 || ids[i] >= ne || !(w[i] > 0.0)) { free(dev_of); return ORC_ROUTING; }
    /* local slot of each expert on its device (placement-list order) */
    int* slot_of = (int*)malloc(sizeof(int) * (size_t)ne);
    for (int d = 0; d < nd; ++d)
        for (int i = 0; i < per; ++i) slot_of[plist[d * per + i]] = i;

    /* source token lists, pipeline.cpp:384-388 */
    int* ntok = (int*)calloc((size_t)(unsigned)nd, sizeof(int));
    for (int t = 0; t < n; ++t) {
        if (sources[t] < 0 || sources[t] >= nd) { free(dev_of); free(slot_of); free(ntok); return ORC_SHAPE; }
        ntok[sources[t]]++;
    }
    int** toks = (int**)malloc(sizeof(int*) * (size_t)nd);
    int** dix = (int**)malloc(sizeof(int*) * (size_t)nd);
    int* nsfd = (int*)calloc((size_t)nd, sizeof(int));
    for (int s = 0; s < nd; ++s) {
        toks[s] = (int*)malloc(sizeof(int) * (size_t)(ntok[s] + 1));
        dix[s] = (int*)malloc(sizeof(int) * (size_t)(nd * ntok[s] + 1));
    }
    {
        int* fill = (int*)calloc((size_t)nd, sizeof(int));
        for (int t = 0; t < n; ++t) toks[sources[t]][fill[sources[t]]++] = t;
        free(fill);
    }
    /* dispatch per source (BRIM0), pipeline.cpp:391-396 */
    long dpos = 0;
    for (int s = 0; s < nd; ++s) {
        nsfd[s] = orc_build_dispatch_index(ids, k, dev_of, nd, toks[s], ntok[s], dix[s]);
        if (dindex_out) {
            memcpy(dindex_out + dpos, dix[s], sizeof(int) * (size_t)nd * ntok[s]);
            dpos += (long)nd * ntok[s];
        }
    }
    /* SFD slot -> token per source (dispatch, pipeline.cpp:109-121) */
    int** sfd_tok = (int**)malloc(sizeof(int*) * (size_t)nd);
    for (int s = 0; s < nd; ++s) {
        sfd_tok[s] = (int*)malloc(sizeof(int) * (size_t)(nsfd[s] + 1));
        for (int d = 0; d < nd; ++d)
            for (int i = 0; i < ntok[s]; ++i) {
                int c = dix[s][(long)d * ntok[s] + i];
                if (c >= 0) sfd_tok[s][c] = toks[s][i];
            }
    }
    /* exchange, pipeline.cpp:125-176: inbox of d ordered (source, counter) */
    long long crossing = 0;
    int* rows_d = (int*)calloc((size_t)nd, sizeof(int));
    for (int s = 0; s < nd; ++s)
        for (int d = 0; d < nd; ++d)
            for (int i = 0; i < ntok[s]; ++i)
                if (dix[s][(long)d * ntok[s] + i] >= 0) rows_d[d]++;
    int** in_tok = (int**)malloc(sizeof(int*) * (size_t)nd);
    int** in_src = (int**)malloc(sizeof(int*) * (size_t)nd);
    int** in_slot = (int**)malloc(sizeof(int*) * (size_t)nd);
    for (int d = 0; d < nd; ++d) {
        in_tok[d] = (int*)malloc(sizeof(int) * (size_t)(rows_d[d] + 1));
        in_src[d] = (int*)malloc(sizeof(int) * (size_t)(rows_d[d] + 1));
        in_slot[d] = (int*)malloc(sizeof(int) * (size_t)(rows_d[d] + 1));
    }
    {
        int* fill = (int*)calloc((size_t)nd, sizeof(int));
        for (int s = 0; s < nd; ++s)
            for (int d = 0; d < nd; ++d)
                for (int i = 0; i < ntok[s]; ++i) {
                    int c = dix[s][(long)d * ntok[s] + i];
                    if (c < 0) continue;
                    int r = fill[d]++;
                    in_tok[d][r] = sfd_tok[s][c];
                    in_src[d][r] = s;
                    in_slot[d][r] = c;
                    if (s != d) ++crossing;
                }
        free(fill);
    }
    /* y_src[s]: nsfd[s] x dm return payloads */
    double** y_src = (double**)malloc(sizeof(double*) * (size_t)nd);
    for (int s = 0; s < nd; ++s) y_src[s] = (double*)calloc((size_t)nsfd[s] * dm + 1, sizeof(double));

    long ipos = 0, cpos = 0;
    for (int d = 0; d < nd; ++d) {
        const int rows = rows_d[d];
        if (inbox_token) {
            memcpy(inbox_token + ipos, in_tok[d], sizeof(int) * (size_t)rows);
            memcpy(inbox_source + ipos, in_src[d], sizeof(int) * (size_t)rows);
            memcpy(inbox_slot + ipos, in_slot[d], sizeof(int) * (size_t)rows);
        }
        ipos += rows;
        /* local ids + weight grid, pipeline.cpp:409-421 */
        char* member = (char*)calloc((size_t)per * rows + 1, 1);
        double* wgrid = (double*)malloc(sizeof(double) * ((size_t)per * rows + 1));
        for (long i = 0; i < (long)per * rows; ++i) wgrid[i] = NAN;
        for (int r = 0; r < rows; ++r) {
            int t = in_tok[d][r];
            for (int j = 0; j < k; ++j) {
                int e = ids[(long)t * k + j];
                if (dev_of[e] != d) continue;
                member[(long)slot_of[e] * rows + r] = 1;
                wgrid[(long)slot_of[e] * rows + r] = w[(long)t * k + j];
            }
        }
        int* cix = (int*)malloc(sizeof(int) * ((size_t)per * rows + 1));
        int n_epd = orc_compute_index_from_member(member, per, rows, cix);
        if (rep) rep->n_epd_dev[d] = n_epd;
        if (cindex_out) { memcpy(cindex_out + cpos, cix, sizeof(int) * (size_t)per * rows); cpos += (long)per * rows; }
        /* scatter -> activation -> modulate -> merge, pipeline.cpp:446-452 */
        double* epd = (double*)malloc(sizeof(double) * ((size_t)n_epd * dh + 1));
        for (int p = 0; p < per; ++p) {
            const int e = plist[d * per + p];
            const double* W1 = w1 + (long)e * dm * dh;
            const double* W3 = w3 ? w3 + (long)e * dm * dh : NULL;
            for (int r = 0; r < rows; ++r) {
                int q = cix[(long)p * rows + r];
                if (q < 0) continue;
                const double* xr = x + (long)in_tok[d][r] * dm;
                const double wt = wgrid[(long)p * rows + r];
                for (int j = 0; j < dh; ++j) {
                    double acc = 0.0;
                    for (int c = 0; c < dm; ++c) acc += xr[c] * W1[(long)c * dh + j];
                    double h = quant(acc, single);
                    if (W3) {
                        double acc3 = 0.0;
                        for (int c = 0; c < dm; ++c) acc3 += xr[c] * W3[(long)c * dh + j];
                        h = quant(quant(act_fn(h, 1), single) * quant(acc3, single), single);
                    } else {
                        h = quant(act_fn(h, act), single);
                    }
                    epd[(long)q * dh + j] = quant(h * wt, single);
                }
            }
        }
        for (int r = 0; r < rows; ++r) {
            double* yo = y_src[in_src[d][r]] + (long)in_slot[d][r] * dm;
            for (int c = 0; c < dm; ++c) {
                double acc = 0.0;
                for (int p = 0; p < per; ++p) {
                    int q = cix[(long)p * rows + r];
                    if (q < 0) continue;
                    const double* W2 = w2 + (long)plist[d * per + p] * dh * dm;
                    for (int j = 0; j < dh; ++j) acc += epd[(long)q * dh + j] * W2[(long)j * dm + c];
                }
                yo[c] = quant(acc, single);
            }
        }
        free(member); free(wgrid); free(cix); free(epd);
    }
    /* combine, pipeline.cpp:285-300 + :470-477 */
    for (int s = 0; s < nd; ++s)
        for (int i = 0; i < ntok[s]; ++i) {
            double* out = x_out + (long)toks[s][i] * dm;
            for (int c = 0; c < dm; ++c) {
                double acc = 0.0;
                for (int d = 0; d < nd; ++d) {
                    int q = dix[s][(long)d * ntok[s] + i];
                    if (q >= 0) acc += y_src[s][(long)q * dm + c];
                }
                out[c] = quant(acc, single);
            }
        }
    /* CommReport, pipeline.cpp:479-487 */
    if (rep) {
        rep->mean_replicas = orc_mean_token_replicas(ids, n, k, dev_of, nd);
        rep->cap_replicas = cap_replicas >= 0.0 ? cap_replicas : (double)(k < nd ? k : nd);
        orc_collaboration_shares(ids, n, k, dev_of, &rep->intra_share, &rep->inter_share);
        rep->crossing_rows = crossing;
        rep->cross_device_bytes = crossing * (long long)dm * bytes_per_scalar;
        for (int d = 0; d < nd; ++d) rep->per_device_rows[d] = rows_d[d];
        for (int s = 0; s < nd; ++s) rep->n_sfd_src[s] = nsfd[s];
    }
    for (int s = 0; s < nd; ++s) { free(toks[s]); free(dix[s]); free(sfd_tok[s]); free(y_src[s]); }
    for (int d = 0; d < nd; ++d) { free(in_tok[d]); free(in_src[d]); free(in_slot[d]); }
    free(toks); free(dix); free(sfd_tok); free(y_src); free(in_tok); free(in_src); free(in_slot);
    free(rows_d); free(nsfd); free(ntok); free(dev_of); free(slot_of);
    return ORC_OK;
}

/* pipeline.cpp:542-562 dense_given_routing (+ the SwiGLU extension when
 * w3 != NULL). Processes only the listed rows (row subsampling: output
 * rows are independent given routing). rows == NULL means all n. */
void orc_dense_given_routing(const double* x, int n, int dm, const int* ids, const double* w, int k,
                             const double* w1, const double* w2, const double* w3, int dh, int act,
                             int single, const int* rows, int nrows, double* out) {
    double* h = (double*)malloc(sizeof(double) * (size_t)dh);
    double* acc = (double*)malloc(sizeof(double) * (size_t)dm);
    const int cnt = rows ? nrows : n;
    for (int ii = 0; ii < cnt; ++ii) {
        const int t = rows ? rows[ii] : ii;
        const double* xr = x + (long)t * dm;
        for (int c = 0; c < dm; ++c) acc[c] = 0.0;
        for (int j = 0; j < k; ++j) {
            const int e = ids[(long)t * k + j];
            const double* W1 = w1 + (long)e * dm * dh;
            const double* W2 = w2 + (long)e * dh * dm;
            for (int q = 0; q < dh; ++q) {
                double a = 0.0;
                for (int c = 0; c < dm; ++c) a += xr[c] * W1[(long)c * dh + q];
                a = quant(a, single);
                if (w3) {
                    const double* W3 = w3 + (long)e * dm * dh;
                    double b = 0.0;
                    for (int c = 0; c < dm; ++c) b += xr[c] * W3[(long)c * dh + q];
                    h[q] = quant(quant(act_fn(a, 1), single) * quant(b, single), single);
                } else {
                    h[q] = quant(act_fn(a, act), single);
                }
            }
            const double wt = w[(long)t * k + j];
            for (int c = 0; c < dm; ++c) {
                double o = 0.0;
                for (int q = 0; q < dh; ++q) o += h[q] * W2[(long)q * dm + c];
                acc[c] += wt * quant(o, single);
            }
        }
        for (int c = 0; c < dm; ++c) out[(long)ii * dm + c] = quant(acc[c], single);
    }
    free(h);
    free(acc);
}

/* Shared (always-active) experts — NOT in the reference; the
 * DeepSeek-MoE / Qwen-MoE extension of BASELINE configs 3 and 5, restated
 * with the same per-expert arithmetic as dense_given_routing above
 * (pipeline.cpp:542-562): for every token t and shared expert s,
 *   h = act(x w1_s)            (2-matrix expert)   or
 *   h = silu(x w1_s) * (x w3_s) (SwiGLU),
 *   y_t += g_t * (h w2_s),  g_t = sigmoid(x_t . gate) if gate, else 1,
 * accumulated in double in ascending s, q, c order and added to out[t]
 * (out is the routed layer output; the product path adds the shared rows
 * last).  Pinned against an independent torch fp64 computation
 * (tests/test_oracle.py::test_shared_experts_oracle_vs_torch).
 *   w1, w3: ns x dm x dh, w2: ns x dh x dm, gate: dm or NULL. */
void orc_shared_experts(const double* x, int n, int dm, const double* w1, const double* w2, const double* w3,
                        int ns, int dh, int act, const double* gate, double* out) {
    double* h = (double*)malloc(sizeof(double) * (size_t)dh);
    double* acc = (double*)malloc(sizeof(double) * (size_t)dm);
    for (int t = 0; t < n; ++t) {
        const double* xr = x + (long)t * dm;
        double g = 1.0;
        if (gate) {
            double z = 0.0;
            for (int c = 0; c < dm; ++c) z += xr[c] * gate[c];
            g = 1.0 / (1.0 + exp(-z));
        }
        for (int c = 0; c < dm; ++c) acc[c] = 0.0;
        for (int s = 0; s < ns; ++s) {
            const double* W1 = w1 + (long)s * dm * dh;
            const double* W2 = w2 + (long)s * dh * dm;
            for (int q = 0; q < dh; ++q) {
                double a = 0.0;
                for (int c = 0; c < dm; ++c) a += xr[c] * W1[(long)c * dh + q];
                if (w3) {
                    const double* W3 = w3 + (long)s * dm * dh;
                    double b = 0.0;
                    for (int c = 0; c < dm; ++c) b += xr[c] * W3[(long)c * dh + q];
                    h[q] = act_fn(a, 1) * b;
                } else {
                    h[q] = act_fn(a, act);
                }
            }
            for (int c = 0; c < dm; ++c) {
                double o = 0.0;
                for (int q = 0; q < dh; ++q) o += h[q] * W2[(long)q * dm + c];
                acc[c] += o;
            }
        }
        for (int c = 0; c < dm; ++c) out[(long)t * dm + c] += g * acc[c];
    }
    free(h);
    free(acc);
}

/* dense_given_routing (pipeline.cpp:542-562) + the shared-expert restatement
 * (orc_shared_experts above) for a SAMPLE of rows, with every operand given
 * in the product's bf16 storage (uint16 bit patterns, widened exactly to
 * double) so the BASELINE-size layers (Mixtral: 8 x 3 x 4096 x 14336 weights)
 * fit in host memory.  Arithmetic is that of orc_dense_given_routing /
 * orc_shared_experts in Precision::Double: per row, experts in routing order,
 * h[q] = act(sum_c x w1) (or silu(sum_c x w1) * sum_c x w3), o[c] = sum_q h w2,
 * acc[c] += w * o[c]; then + g * sum_s FFN_s.  The loops are blocked over the
 * sampled rows so each weight row is read once per expert for all of them;
 * every per-element sum keeps the ascending order of the scalar version.
 * Rows are independent given routing (pipeline.cpp:548-560), so a sample is a
 * valid full-size check.  rows[nrows] index into x [n, dm]; ids/w [n, k];
 * w1/w3 [E, dm, dh], w2 [E, dh, dm]; shared (ns > 0): w1s/w3s [ns, dm, dhs],
 * w2s [ns, dhs, dm], gate_s [dm] or NULL.  out [nrows, dm]. */
static inline double bf(uint16_t v) {
    union { uint32_t u; float f; } c;
    c.u = (uint32_t)v << 16;
    return (double)c.f;
}
static void ffn_rows_bf16(const double* xr, int nr, int dm, const uint16_t* W1, const uint16_t* W3, const uint16_t* W2,
                          int dh, int act, const double* scale, double* acc) {
    /* xr [nr, dm] doubles; acc[r, c] += scale[r] * (h_r W2)[c] */
    double* a = (double*)calloc((size_t)nr * dh, sizeof(double));
    double* b = W3 ? (double*)calloc((size_t)nr * dh, sizeof(double)) : NULL;
    double* wrow = (double*)malloc(sizeof(double) * (size_t)dh);
    for (int c = 0; c < dm; ++c) { /* ascending c for every (r, q) */
        for (int q = 0; q < dh; ++q) wrow[q] = bf(W1[(long)c * dh + q]);
        for (int r = 0; r < nr; ++r) {
            const double xv = xr[(long)r * dm + c];
            double* ar = a + (long)r * dh;
            for (int q = 0; q < dh; ++q) ar[q] += xv * wrow[q];
        }
        if (W3) {
            for (int q = 0; q < dh; ++q) wrow[q] = bf(W3[(long)c * dh + q]);
            for (int r = 0; r < nr; ++r) {
                const double xv = xr[(long)r * dm + c];
                double* br = b + (long)r * dh;
                for (int q = 0; q < dh; ++q) br[q] += xv * wrow[q];
            }
        }
    }
    for (long i = 0; i < (long)nr * dh; ++i) a[i] = W3 ? act_fn(a[i], 1) * b[i] : act_fn(a[i], act);
    double* o = (double*)calloc((size_t)nr * dm, sizeof(double));
    double* w2row = (double*)malloc(sizeof(double) * (size_t)dm);
    for (int q = 0; q < dh; ++q) { /* ascending q for every (r, c) */
        for (int c = 0; c < dm; ++c) w2row[c] = bf(W2[(long)q * dm + c]);
        for (int r = 0; r < nr; ++r) {
            const double hv = a[(long)r * dh + q];
            double* orow = o + (long)r * dm;
            for (int c = 0; c < dm; ++c) orow[c] += hv * w2row[c];
        }
    }
    for (int r = 0; r < nr; ++r)
        for (int c = 0; c < dm; ++c) acc[(long)r * dm + c] += scale[r] * o[(long)r * dm + c];
    free(a);
    free(b);
    free(wrow);
    free(o);
    free(w2row);
}

void orc_dense_rows_bf16(const uint16_t* x, int n, int dm, const int* ids, const float* w, int k, int ne,
                         const uint16_t* w1, const uint16_t* w2, const uint16_t* w3, int dh, int act,
                         int ns, const uint16_t* w1s, const uint16_t* w2s, const uint16_t* w3s, int dhs,
                         const uint16_t* gate_s, const int* rows, int nrows, double* out) {
    (void)n;
    double* xr = (double*)malloc(sizeof(double) * (size_t)nrows * dm);
    double* sub = (double*)malloc(sizeof(double) * (size_t)nrows * dm);
    double* acc = (double*)calloc((size_t)nrows * dm, sizeof(double));
    double* sc = (double*)malloc(sizeof(double) * (size_t)nrows);
    int* pick = (int*)malloc(sizeof(int) * (size_t)nrows);
    for (int r = 0; r < nrows; ++r)
        for (int c = 0; c < dm; ++c) xr[(long)r * dm + c] = bf(x[(long)rows[r] * dm + c]);
    /* routed experts: slot j of every row in routing order (acc[c] += w o[c]
     * in slot order per row, like the scalar version); rows sharing an expert
     * in slot j are batched */
    for (int j = 0; j < k; ++j)
        for (int e = 0; e < ne; ++e) {
            int m = 0;
            for (int r = 0; r < nrows; ++r)
                if (ids[(long)rows[r] * k + j] == e) pick[m++] = r;
            if (!m) continue;
            for (int i = 0; i < m; ++i) {
                memcpy(sub + (long)i * dm, xr + (long)pick[i] * dm, sizeof(double) * dm);
                sc[i] = (double)w[(long)rows[pick[i]] * k + j];
            }
            double* tmp = (double*)calloc((size_t)m * dm, sizeof(double));
            ffn_rows_bf16(sub, m, dm, w1 + (long)e * dm * dh, w3 ? w3 + (long)e * dm * dh : NULL,
                          w2 + (long)e * dh * dm, dh, act, sc, tmp);
            for (int i = 0; i < m; ++i)
                for (int c = 0; c < dm; ++c) acc[(long)pick[i] * dm + c] += tmp[(long)i * dm + c];
            free(tmp);
        }
    if (ns > 0) {
        double* sh = (double*)calloc((size_t)nrows * dm, sizeof(double));
        for (int r = 0; r < nrows; ++r) sc[r] = 1.0;
        for (int s2 = 0; s2 < ns; ++s2)
            ffn_rows_bf16(xr, nrows, dm, w1s + (long)s2 * dm * dhs, w3s ? w3s + (long)s2 * dm * dhs : NULL,
                          w2s + (long)s2 * dhs * dm, dhs, act, sc, sh);
        for (int r = 0; r < nrows; ++r) {
            double g = 1.0;
            if (gate_s) {
                double z = 0.0;
                for (int c = 0; c < dm; ++c) z += xr[(long)r * dm + c] * bf(gate_s[c]);
                g = 1.0 / (1.0 + exp(-z));
            }
            for (int c = 0; c < dm; ++c) acc[(long)r * dm + c] += g * sh[(long)r * dm + c];
        }
        free(sh);
    }
    memcpy(out, acc, sizeof(double) * (size_t)nrows * dm);
    free(xr);
    free(sub);
    free(acc);
    free(sc);
    free(pick);
}

/* matrix.cpp:52-60 */
double orc_max_rel_error(const double* a, const double* b, long n) {
    double diff = 0.0, ref = 0.0;
    for (long i = 0; i < n; ++i) {
        double dd = fabs(a[i] - b[i]);
        if (dd > diff) diff = dd;
        if (fabs(b[i]) > ref) ref = fabs(b[i]);
    }
    return diff / (ref > 1e-300 ? ref : 1e-300);
}
