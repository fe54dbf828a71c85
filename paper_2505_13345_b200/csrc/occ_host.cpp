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
