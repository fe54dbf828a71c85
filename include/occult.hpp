// occult.hpp — header-only C++ host mirror of the reference API over the C-ABI
// (occult.h).  Same names, argument meaning and error behaviour as namespace
// moesim (/root/reference/proj/include/moesim/*.hpp); buffers are device
// pointers (bf16 tokens/experts, int32 ids, f32 weights) and every call is
// ordered on a CUDA stream.  Errors are thrown as the reference's exception
// types (common.hpp:11-34), translated from occ_status.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "occult.h"

namespace occult {

struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PlacementError : std::runtime_error { using std::runtime_error::runtime_error; };
struct RoutingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(occ_status s, const char* what) {
    if (s == OCC_OK) return;
    const std::string msg = std::string(what) + ": " + occ_last_error();
    switch (s) {
        case OCC_ERR_SHAPE: throw ShapeError(msg);
        case OCC_ERR_CONFIG: throw ConfigError(msg);
        case OCC_ERR_PLACEMENT: throw PlacementError(msg);
        case OCC_ERR_ROUTING: throw RoutingError(msg);
        case OCC_ERR_CAPACITY: throw CapacityError(msg);
        case OCC_ERR_STATE: throw StateError(msg);
        default: throw DeviceError(msg);
    }
}

// moesim::Placement (placement.hpp:14-25): per-device expert lists.
struct Placement {
    std::vector<std::vector<int>> devices;
    int num_devices() const { return static_cast<int>(devices.size()); }
    std::vector<int32_t> flat() const {
        std::vector<int32_t> f;
        for (const auto& d : devices) f.insert(f.end(), d.begin(), d.end());
        return f;
    }
};

inline Placement trivial_placement(int num_experts, int num_devices) {  // placement.cpp:47-58
    if (num_devices < 1 || num_experts < 1 || num_experts % num_devices)
        throw ConfigError("trivial_placement: num_experts must be a positive multiple of num_devices");
    Placement p;
    const int per = num_experts / num_devices;
    p.devices.resize(num_devices);
    for (int d = 0; d < num_devices; ++d)
        for (int i = 0; i < per; ++i) p.devices[d].push_back(d * per + i);
    return p;
}

// moesim::reschedule_placement (placement.cpp:88-148), host, bit-exact.
inline Placement reschedule_placement(const std::vector<double>& norm_graph, int num_experts, int num_devices) {
    std::vector<int32_t> flat(num_experts);
    check(occ_reschedule_placement(norm_graph.data(), num_experts, num_devices, flat.data()), "reschedule_placement");
    Placement p;
    const int per = num_experts / num_devices;
    for (int d = 0; d < num_devices; ++d) p.devices.emplace_back(flat.begin() + d * per, flat.begin() + (d + 1) * per);
    return p;
}

struct CommReport {  // moesim::CommReport (collab.hpp:36-43)
    double mean_replicas = 0, cap_replicas = 0, intra_share = 0, inter_share = 0;
    long long cross_device_bytes = 0, naive_crossing_rows = 0;
    std::vector<long long> per_device_token_counts;
};

// One GPU's share of the EP layer: router config + placement + resident experts.
class Layer {
  public:
    Layer(const occ_config& cfg, const Placement& placement, int world_size = 1, int rank = 0) : cfg_(cfg) {
        const auto flat = placement.flat();
        if (static_cast<int>(flat.size()) != cfg.num_experts)
            throw PlacementError("placement: covers " + std::to_string(flat.size()) + " experts");
        check(occ_create(&cfg, flat.data(), world_size, rank, &h_), "occ_create");
    }
    ~Layer() { occ_destroy(h_); }
    Layer(const Layer&) = delete;
    Layer& operator=(const Layer&) = delete;

    occ_handle* handle() const { return h_; }

    // Reference layout (token.hpp:30-44): w1/w3 [E_l, D, F], w2 [E_l, F, D], bf16, device.
    void load_experts(const void* w1, const void* w2, const void* w3, occ_stream_t s) {
        check(occ_load_experts(h_, w1, w3, w2, s), "load_experts");
    }
    // DeepSeek / Qwen shared experts (not in the reference): w1/w3 [S, D, F_s], w2 [S, F_s, D],
    // gate [D] or nullptr; num_shared = 0 detaches them.
    void load_shared_experts(int num_shared, int d_ff_shared, const void* w1, const void* w2, const void* w3,
                             const void* gate, occ_stream_t s) {
        check(occ_load_shared_experts(h_, num_shared, d_ff_shared, w1, w3, w2, gate, s), "load_shared_experts");
    }
    void set_validate(bool on) { check(occ_set_validate(h_, on), "set_validate"); }
    // Two micro-batches per forward on two streams (exchange / GEMM overlap); collective at world > 1.
    void set_micro_batches(int micro_batches, int comm_sms = -1) {
        check(occ_set_micro_batches(h_, micro_batches, comm_sms), "set_micro_batches");
    }
    void set_placement(const Placement& placement) {
        std::vector<int32_t> flat;
        for (const auto& d : placement.devices) flat.insert(flat.end(), d.begin(), d.end());
        check(occ_set_placement(h_, flat.data()), "set_placement");
    }
    // Training: keep what backward_vjps (backward.cpp:24-161) needs; call before load_experts.
    void set_training(bool on) { check(occ_set_training(h_, on), "set_training"); }
    void backward(const void* upstream, float* g_x, float* g_w1, float* g_w3, float* g_w2, float* g_weights,
                  occ_stream_t s) {
        check(occ_backward(h_, upstream, g_x, g_w1, g_w3, g_w2, g_weights, s), "backward");
    }
    // End to end from pinned host memory (copies overlapped with the neighbouring calls).
    void forward_host(const void* x_host, const void* gate, const occ_prune* prune, int n, void* out_host,
                      occ_stream_t s) {
        check(occ_forward_host(h_, x_host, gate, prune, n, out_host, 1, s), "forward_host");
    }
    void host_wait(occ_stream_t s) { check(occ_host_wait(h_, s), "host_wait"); }

    // forward_given_routing (pipeline.cpp:360-501)
    void forward_given_routing(const void* x, const int32_t* ids, const float* w, const int32_t* sources, int n,
                               void* out, occ_stream_t s) {
        check(occ_forward(h_, x, ids, w, sources, n, out, s), "forward_given_routing");
    }
    // forward_expert_parallel (pipeline.cpp:503-517)
    void forward_expert_parallel(const void* x, const void* gate, const occ_prune* prune, const int32_t* sources,
                                 int n, void* out, occ_stream_t s) {
        check(occ_forward_expert_parallel(h_, x, gate, prune, sources, n, out, s), "forward_expert_parallel");
    }
    // Router arithmetic: OCC_ROUTER_TC (default) or OCC_ROUTER_EXACT (the
    // reference's gate_scores + topk_route + prune_routing, bit-exact).
    void set_router_mode(int mode) { check(occ_set_router_mode(h_, mode), "set_router_mode"); }
    // gate_scores -> topk_route -> prune_routing (routing.cpp:33-84,
    // pruning.cpp:141-163) on bf16 tokens / gate, bit-exact: ids int32, weights f64.
    void route_exact(const void* x, const void* gate, int n, const occ_prune* prune, int32_t* ids, double* weights,
                     double* scores, occ_stream_t s) {
        check(occ_route_exact(h_, x, gate, n, prune, ids, weights, scores, s), "route_exact");
    }

    // ---- stage-level entry points (pipeline.hpp:89-123) ----
    // build_dispatch_index: world_size 1 -> every source (sources nullable), BRIM0s
    // concatenated + counts [N_d x N_d]; world_size > 1 -> this rank's tokens.
    void build_dispatch_index(const int32_t* ids, const int32_t* sources, int n, int32_t* brim0, int32_t* counts,
                              occ_stream_t s) {
        check(occ_build_dispatch(h_, ids, sources, n, brim0, counts, s), "build_dispatch_index");
    }
    // dispatch (pipeline.cpp:91-123): one source's SfdBatch from its BRIM0 [N_d x n].
    void dispatch(const void* x, const int32_t* ids, const float* w, int n, const int32_t* brim0, void* sfd_x,
                  int32_t* sfd_ids, float* sfd_w, int32_t* sfd_token, occ_stream_t s) {
        check(occ_dispatch(h_, x, ids, w, n, brim0, sfd_x, sfd_ids, sfd_w, sfd_token, s), "dispatch");
    }
    // build_compute_index (pipeline.cpp:52-89) of EP device `device` over its inbox rows.
    void build_compute_index(int device, const int32_t* in_ids, const float* in_w, int rows, int32_t* cindex,
                             int32_t* n_epd, occ_stream_t s) {
        check(occ_build_compute(h_, device, in_ids, in_w, rows, cindex, n_epd, s), "build_compute_index");
    }
    // scatter_matmul -> apply_activation -> weight_modulate -> merge_matmul
    // (pipeline.cpp:178-283): the partial-combined return rows of device `device`.
    void expert_compute(int device, const void* in_x, const int32_t* in_ids, const float* in_w, int rows, void* y,
                        occ_stream_t s) {
        check(occ_expert_compute(h_, device, in_x, in_ids, in_w, rows, y, s), "expert_compute");
    }
    // combine (pipeline.cpp:285-300) of one source through its BRIM0.
    void combine(const void* y_returned, const int32_t* brim0, int n, void* out, occ_stream_t s) {
        check(occ_combine(h_, y_returned, brim0, n, out, s), "combine");
    }

    CommReport report(int bytes_per_scalar, occ_stream_t s) const {
        occ_comm_report r{};
        check(occ_comm_report_get(h_, bytes_per_scalar, &r, s), "comm_report");
        CommReport c{r.mean_replicas, r.cap_replicas, r.intra_share, r.inter_share, r.cross_device_bytes,
                     r.naive_crossing_rows, {}};
        for (int d = 0; d < cfg_.num_devices; ++d) c.per_device_token_counts.push_back(r.per_device_rows[d]);
        return c;
    }

  private:
    occ_config cfg_;
    occ_handle* h_ = nullptr;
};

}  // namespace occult
