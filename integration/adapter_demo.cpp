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
    try {
        ParallelPlan bad = plan;
        bad.avg_frequency = 0;
        b200::train_parallel(bad, m0, tr, cv, opts, o);
    } catch (const Error& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
    }
    return 0;
}
