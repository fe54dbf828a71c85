// moesim_gpu.hpp — the reference-side binding a moesim maintainer adds to
// route forward_given_routing / forward_expert_parallel / build_dispatch_index
// through the B200 library.  Same signatures as pipeline.hpp:83-84 and
// :178-189 and the same exception types; moesim's host Matrix values are
// converted to bf16 device buffers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <span>
#include <vector>

#include "moesim/pipeline.hpp"
#include "occult.hpp"

namespace moesim_gpu {

namespace detail {

inline void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

template <class T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
};

inline std::vector<__nv_bfloat16> to_bf16(const std::vector<double>& v) {
    std::vector<__nv_bfloat16> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = __float2bfloat16(static_cast<float>(v[i]));
    return o;
}

inline occ_config config_of(const moesim::MoEConfig& c) {
    return occ_config{c.num_experts, c.top_k, c.num_devices, c.embed_dim, c.hidden_dim, c.renormalize ? 1 : 0,
                      static_cast<int>(c.activation), 1};
}

// occult errors -> the reference's own exception types (common.hpp:11-34)
template <class F>
auto translate(F&& f) {
    try {
        return f();
    } catch (const occult::ShapeError& e) { throw moesim::ShapeError(e.what());
    } catch (const occult::ConfigError& e) { throw moesim::ConfigError(e.what());
    } catch (const occult::PlacementError& e) { throw moesim::PlacementError(e.what());
    } catch (const occult::RoutingError& e) { throw moesim::RoutingError(e.what());
    } catch (const occult::CapacityError& e) { throw moesim::CapacityError(e.what());
    } catch (const occult::StateError& e) { throw moesim::StateError(e.what()); }
}

}  // namespace detail

// moesim::forward_given_routing (pipeline.hpp:178-182) on the B200.
inline moesim::ForwardResult forward_given_routing(const moesim::TokenMatrix& x, const moesim::RoutingOutcome& routing,
                                                   const moesim::ExpertWeights& experts,
                                                   const moesim::Placement& placement,
                                                   const moesim::MoEConfig& config, std::span<const int> sources = {},
                                                   int bytes_per_scalar = 4, double cap_replicas = -1.0) {
    using namespace detail;
    return translate([&] {
        config.validate();
        placement.validate(config.num_experts);
        if (x.rows() != routing.num_tokens) throw moesim::ShapeError("forward: routing token count mismatch");
        const int n = x.rows(), D = config.embed_dim, F = config.hidden_dim, E = config.num_experts, k = routing.k;
        occult::Placement pl{placement.devices};
        occult::Layer layer(config_of(config), pl);
        cudaStream_t st = nullptr;
        // experts in reference layout: w1 [E, D, F], w2 [E, F, D]
        std::vector<double> w1, w2;
        for (int e = 0; e < E; ++e) {
            w1.insert(w1.end(), experts.w1[e].data.begin(), experts.w1[e].data.end());
            w2.insert(w2.end(), experts.w2[e].data.begin(), experts.w2[e].data.end());
        }
        const auto w1b = to_bf16(w1), w2b = to_bf16(w2), xb = to_bf16(x.values.data);
        Dev<__nv_bfloat16> dw1(w1b.size()), dw2(w2b.size()), dx(xb.size()), dout(xb.size());
        Dev<int32_t> dids((size_t)n * k), dsrc(n);
        Dev<float> dw((size_t)n * k);
        std::vector<float> wf(routing.weights.begin(), routing.weights.end());
        cuda_check(cudaMemcpy(dw1.p, w1b.data(), w1b.size() * 2, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dw2.p, w2b.data(), w2b.size() * 2, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dx.p, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dids.p, routing.ids.data(), sizeof(int) * n * k, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dw.p, wf.data(), sizeof(float) * n * k, cudaMemcpyHostToDevice));
        if (!sources.empty()) cuda_check(cudaMemcpy(dsrc.p, sources.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
        layer.load_experts(dw1.p, dw2.p, nullptr, st);
        layer.forward_given_routing(dx.p, dids.p, dw.p, sources.empty() ? nullptr : dsrc.p, n, dout.p, st);
        std::vector<__nv_bfloat16> ob(xb.size());
        cuda_check(cudaMemcpy(ob.data(), dout.p, ob.size() * 2, cudaMemcpyDeviceToHost));
        moesim::ForwardResult res;
        res.x_out = moesim::TokenMatrix(moesim::Matrix(n, D), moesim::TokenState::Ori);
        for (size_t i = 0; i < ob.size(); ++i) res.x_out.values.data[i] = __bfloat162float(ob[i]);
        const occult::CommReport r = layer.report(bytes_per_scalar, st);
        res.report.mean_replicas = r.mean_replicas;
        res.report.cap_replicas =
            cap_replicas >= 0.0 ? cap_replicas : static_cast<double>(std::min(k, config.num_devices));
        res.report.intra_share = r.intra_share;
        res.report.inter_share = r.inter_share;
        res.report.cross_device_bytes = r.cross_device_bytes;
        res.report.per_device_token_counts = r.per_device_token_counts;
        (void)F;
        return res;
    });
}

// moesim::build_dispatch_index (pipeline.hpp:83-84) for one source's tokens
// (ascending Ori rows) on the B200: the BRIM0 counters, bit-exact.
inline moesim::DispatchIndex build_dispatch_index(const moesim::RoutingOutcome& routing,
                                                  const moesim::Placement& placement, std::span<const int> tokens) {
    using namespace detail;
    return translate([&] {
        const int nd = placement.num_devices(), k = routing.k, n = static_cast<int>(tokens.size());
        int ne = 0;
        for (const auto& d : placement.devices) ne += static_cast<int>(d.size());
        occ_config cfg{ne, k, nd, 8, 8, 1, 0, 1};
        occult::Layer layer(cfg, occult::Placement{placement.devices});
        std::vector<int32_t> ids((size_t)n * k), src(n, 0);  // all rows: one source
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < k; ++j) ids[(size_t)i * k + j] = routing.ids[(size_t)tokens[i] * k + j];
        Dev<int32_t> dids(ids.size()), dsrc(n), db((size_t)nd * n), dc((size_t)nd * nd);
        cuda_check(cudaMemcpy(dids.p, ids.data(), sizeof(int32_t) * ids.size(), cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dsrc.p, src.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
        layer.build_dispatch_index(dids.p, dsrc.p, n, db.p, dc.p, nullptr);
        moesim::DispatchIndex di;
        di.num_devices = nd;
        di.num_tokens = n;
        di.entries.resize((size_t)nd * n);
        cuda_check(cudaMemcpy(di.entries.data(), db.p, sizeof(int32_t) * di.entries.size(), cudaMemcpyDeviceToHost));
        di.n_sfd = 0;
        for (int v : di.entries) di.n_sfd += v >= 0;
        return di;
    });
}

// moesim::forward_expert_parallel (pipeline.hpp:185-189) on the B200 with the
// exact router: gate_scores + topk_route (+ prune_routing) bit-exact with the
// reference, then the indexed data path.
inline moesim::ForwardResult forward_expert_parallel(const moesim::TokenMatrix& x, const moesim::GateMatrix& gate,
                                                     const moesim::ExpertWeights& experts,
                                                     const moesim::Placement& placement,
                                                     const moesim::PruneSpec& prune,
                                                     const moesim::MoEConfig& config,
                                                     std::span<const int> sources = {}, int bytes_per_scalar = 4) {
    using namespace detail;
    moesim::RoutingOutcome routing = translate([&] {
        config.validate();
        const int n = x.rows(), D = config.embed_dim, E = config.num_experts, k = config.top_k;
        occult::Layer layer(config_of(config), occult::Placement{placement.devices});
        const auto xb = to_bf16(x.values.data), gb = to_bf16(gate.weights.data);
        Dev<__nv_bfloat16> dx(xb.size()), dg(gb.size());
        Dev<int32_t> dids((size_t)n * k);
        Dev<double> dw((size_t)n * k);
        cuda_check(cudaMemcpy(dx.p, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dg.p, gb.data(), gb.size() * 2, cudaMemcpyHostToDevice));
        occ_prune pr{static_cast<int>(prune.mode), prune.device_budget,
                     prune.weight_policy == moesim::ReplacementWeightPolicy::OwnScore ? 1 : 0};
        if (prune.mode == moesim::PruneMode::Similarity) throw moesim::ConfigError("binding: router-score pruning only");
        layer.route_exact(dx.p, dg.p, n, prune.mode == moesim::PruneMode::None ? nullptr : &pr, dids.p, dw.p, nullptr,
                          nullptr);
        moesim::RoutingOutcome r;
        r.num_tokens = n;
        r.k = k;
        r.ids.resize((size_t)n * k);
        r.weights.resize((size_t)n * k);
        cuda_check(cudaMemcpy(r.ids.data(), dids.p, sizeof(int32_t) * r.ids.size(), cudaMemcpyDeviceToHost));
        cuda_check(cudaMemcpy(r.weights.data(), dw.p, sizeof(double) * r.weights.size(), cudaMemcpyDeviceToHost));
        (void)D;
        (void)E;
        return r;
    });
    double cap = static_cast<double>(std::min(config.top_k, placement.num_devices()));
    if (prune.mode != moesim::PruneMode::None) cap = std::min(cap, static_cast<double>(prune.device_budget));
    return moesim_gpu::forward_given_routing(x, routing, experts, placement, config, sources, bytes_per_scalar, cap);
}

}  // namespace moesim_gpu
