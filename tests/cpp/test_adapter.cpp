// Reference-side check of the drop-in: the same inputs through
// moesim::forward_given_routing (reference, CPU) and
// moesim_gpu::forward_given_routing (B200 via libocc.so).  Exit 0 on pass.
#include <cmath>
#include <cstdio>

#include "moesim/pipeline.hpp"
#include "moesim/pruning.hpp"
#include "moesim/routing.hpp"
#include "moesim_gpu.hpp"

using namespace moesim;

static double bf16r(double v) { return __bfloat162float(__float2bfloat16(static_cast<float>(v))); }

int main() {
    int fails = 0;
    for (int nd : {1, 2, 4}) {
        MoEConfig cfg;
        cfg.num_experts = 8;
        cfg.top_k = 2;
        cfg.num_devices = nd;
        cfg.embed_dim = 64;
        cfg.hidden_dim = 128;
        cfg.precision = Precision::Double;
        cfg.activation = Activation::SiLU;
        Rng master(1);
        Rng token_rng(master.next()), gate_rng(master.next()), expert_rng(master.next());
        TokenMatrix x(random_matrix(300, 64, token_rng, Precision::Double), TokenState::Ori);
        ExpertWeights ex = ExpertWeights::random(8, 64, 128, expert_rng, Precision::Double, Activation::SiLU);
        GateMatrix gate{random_matrix(8, 64, gate_rng, Precision::Double)};
        for (double& v : x.values.data) v = bf16r(v);
        for (double& v : gate.weights.data) v = bf16r(v);  // the device router reads a bf16 gate
        for (auto& m : ex.w1) for (double& v : m.data) v = bf16r(v / 8.0);
        for (auto& m : ex.w2) for (double& v : m.data) v = bf16r(v / std::sqrt(128.0));
        RoutingOutcome r = topk_route(gate_scores(x, gate), 2, true);
        for (double& w : r.weights) w = static_cast<float>(w);
        const Placement p = trivial_placement(8, nd);
        const ForwardResult want = forward_given_routing(x, r, ex, p, cfg);
        const ForwardResult got = moesim_gpu::forward_given_routing(x, r, ex, p, cfg);
        const double err = max_rel_error(got.x_out.values, want.x_out.values);
        const bool ok = err <= 1e-2 && got.report.mean_replicas == want.report.mean_replicas &&
                        got.report.cross_device_bytes == want.report.cross_device_bytes &&
                        got.report.per_device_token_counts == want.report.per_device_token_counts &&
                        got.report.intra_share == want.report.intra_share;
        std::printf("nd=%d max_rel_error=%.3e replicas=%.4f bytes=%lld %s\n", nd, err, got.report.mean_replicas,
                    got.report.cross_device_bytes, ok ? "ok" : "FAIL");
        fails += !ok;
        // error behaviour: a duplicate expert id raises moesim::RoutingError, as in the reference
        RoutingOutcome bad = r;
        bad.ids[1] = bad.ids[0];
        bool threw = false;
        try {
            moesim_gpu::forward_given_routing(x, bad, ex, p, cfg);
        } catch (const RoutingError&) {
            threw = true;
        }
        std::printf("  duplicate id -> moesim::RoutingError: %s\n", threw ? "ok" : "FAIL");
        fails += !threw;
        // build_dispatch_index of one source's tokens: the BRIM0 counters bit for bit
        std::vector<int> tokens;
        for (int t = 1; t < 300; t += 3) tokens.push_back(t);
        const DispatchIndex di_ref = build_dispatch_index(r, p, tokens);
        const DispatchIndex di_gpu = moesim_gpu::build_dispatch_index(r, p, tokens);
        const bool di_ok = di_ref.entries == di_gpu.entries && di_ref.n_sfd == di_gpu.n_sfd;
        std::printf("  build_dispatch_index: %s\n", di_ok ? "ok" : "FAIL");
        fails += !di_ok;
        // forward_expert_parallel with the exact router: routing bit-exact, so the
        // CommReport is identical; values within the bf16 tolerance
        PruneSpec none;
        const ForwardResult fe_ref = forward_expert_parallel(x, gate, ex, p, none, cfg);
        const ForwardResult fe_gpu = moesim_gpu::forward_expert_parallel(x, gate, ex, p, none, cfg);
        const double fe_err = max_rel_error(fe_gpu.x_out.values, fe_ref.x_out.values);
        const bool fe_ok = fe_err <= 1e-2 && fe_gpu.report.mean_replicas == fe_ref.report.mean_replicas &&
                           fe_gpu.report.cross_device_bytes == fe_ref.report.cross_device_bytes &&
                           fe_gpu.report.per_device_token_counts == fe_ref.report.per_device_token_counts &&
                           fe_gpu.report.intra_share == fe_ref.report.intra_share &&
                           fe_gpu.report.cap_replicas == fe_ref.report.cap_replicas;
        std::printf("  forward_expert_parallel (exact router): max_rel_error=%.3e %s\n", fe_err, fe_ok ? "ok" : "FAIL");
        fails += !fe_ok;
        if (nd >= 2) {  // with router-score pruning to one device per token
            PruneSpec pr;
            pr.mode = PruneMode::RouterScore;
            pr.device_budget = 1;
            const ForwardResult pp_ref = forward_expert_parallel(x, gate, ex, p, pr, cfg);
            const ForwardResult pp_gpu = moesim_gpu::forward_expert_parallel(x, gate, ex, p, pr, cfg);
            const bool pp_ok = max_rel_error(pp_gpu.x_out.values, pp_ref.x_out.values) <= 1e-2 &&
                               pp_gpu.report.mean_replicas == pp_ref.report.mean_replicas &&
                               pp_gpu.report.cross_device_bytes == pp_ref.report.cross_device_bytes;
            std::printf("  forward_expert_parallel (router pruning, budget 1): %s\n", pp_ok ? "ok" : "FAIL");
            fails += !pp_ok;
        }
    }
    std::printf(fails ? "ADAPTER FAIL\n" : "ADAPTER OK\n");
    return fails;
}
