// Drop-in demo: the reference's own types and train_parallel (linked from the
// reference objects in oracle/_ref) next to the B200 adapter, on the same
// inputs. Prints one JSON line with both results. Built by integration/Makefile.
#include <cmath>
#include <cstdio>

#include "parnn/rng.hpp"
#include "parnn_reference_adapter.hpp"

int main() {
    using namespace parnn;
    Dataset all = generate_synthetic(10, 12, 20, 4.0, 1);
    SplitSpec spec;
    spec.cv_fraction = 0.1;
    spec.seed = 2;
    auto [tr, cv] = split_cv(all, spec);
    const FeatureStats st = feature_stats(tr);
    standardize_in_place(tr, st);
    standardize_in_place(cv, st);
    Rng rng(3);
    const MlpModel m0 = init_random({12, 16, 14, 10}, Activation::sigmoid, rng);
    ParallelPlan plan;
    plan.workers = 4;
    plan.avg_frequency = 2;
    plan.minibatch = 8;
    plan.base_seed = 17;
    TrainOptions opts;
    opts.optimizer = OptimizerKind::ngsgd;
    opts.epochs = 2;
    const TrainResult ref = train_parallel(plan, m0, tr, cv, opts);
    b200::Options o;
    o.precision = PARNN_FP32;
    const TrainResult ours = b200::train_parallel(plan, m0, tr, cv, opts, o);
    const ParamVector a = flatten(ref.model), b = flatten(ours.model);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
        den += a.data[i] * a.data[i];
    }
    std::printf("{\"epochs\": [%zu, %zu], \"ce_ref\": %.9f, \"ce_b200\": %.9f, \"theta_rel_l2\": %.3e, "
                "\"avg_events\": [%zu, %zu]}\n",
                ref.metrics.size(), ours.metrics.size(), ref.metrics.back().train_ce, ours.metrics.back().train_ce,
                std::sqrt(num / den), ref.metrics.back().avg_events, ours.metrics.back().avg_events);
    // the north star's low-rank NG-SGD through the same adapter call
    b200::Options lo = o;
    lo.lowrank_ng = true;
    const TrainResult low = b200::train_parallel(plan, m0, tr, cv, opts, lo);
    std::printf("{\"lowrank_epochs\": %zu, \"ce_lowrank\": %.9f, \"ce_ref\": %.9f}\n", low.metrics.size(),
                low.metrics.back().train_ce, ref.metrics.back().train_ce);
    // greedy_pretrain on the caller's Rng: the reference and the adapter leave their
    // Rng in the same state and produce bit-identical output layers
    {
        const std::vector<std::size_t> pdims{12, 10, 8, 10};
        PretrainOptions po;
        po.epochs = 2;
        po.batch_size = 8;
        Matrix data(64, 12);
        for (std::size_t i = 0; i < 64; ++i)
            for (std::size_t j = 0; j < 12; ++j) data(i, j) = tr.features(i, j);
        Rng ra(41), rb(41);
        ra.gaussian(0.0, 1.0);  // leave a cached polar spare in both: it must cross the ABI too
        rb.gaussian(0.0, 1.0);
        const MlpModel pa = greedy_pretrain(pdims, data, po, Activation::sigmoid, ra);
        const MlpModel pb = b200::greedy_pretrain(pdims, data, po, Activation::sigmoid, rb);
        const auto& wa = pa.layers.back().weights.data();
        const auto& wb = pb.layers.back().weights.data();
        bool out_equal = wa.size() == wb.size();
        for (std::size_t i = 0; out_equal && i < wa.size(); ++i) out_equal = wa[i] == wb[i];
        bool rng_equal = true;
        for (int i = 0; i < 8; ++i) rng_equal = rng_equal && ra.next_u64() == rb.next_u64();
        rng_equal = rng_equal && ra.gaussian(0.0, 1.0) == rb.gaussian(0.0, 1.0);
        double num = 0, den = 0;
        const auto& la = pa.layers[0].weights.data();
        const auto& lb = pb.layers[0].weights.data();
        for (std::size_t i = 0; i < la.size(); ++i) {
            num += (la[i] - lb[i]) * (la[i] - lb[i]);
            den += la[i] * la[i];
        }
        std::printf("{\"pretrain_output_layer_equal\": %s, \"pretrain_rng_state_equal\": %s, "
                    "\"pretrain_layer0_rel_l2\": %.3e, \"activation_equal\": %s}\n",
                    out_equal ? "true" : "false", rng_equal ? "true" : "false", std::sqrt(num / den),
                    pa.activation == pb.activation ? "true" : "false");
    }
    try {
        ParallelPlan bad = plan;
        bad.avg_frequency = 0;
        b200::train_parallel(bad, m0, tr, cv, opts, o);
    } catch (const Error& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
    }
    return 0;
}
