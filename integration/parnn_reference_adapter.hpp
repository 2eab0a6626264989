// Reference-side adapter: the parnn C++ API (namespace parnn, reference
// headers parallel.hpp / network.hpp / pretrain.hpp) implemented on top of the
// B200 C ABI (include/parnn_b200.h). A maintainer of the reference swaps the
// body of parnn::train_parallel / serial_train / greedy_pretrain
// (parallel.cpp:279-294, pretrain.cpp:162-207) for these calls; every value
// type stays the reference's own, and errors come back as parnn::Error with
// the reference's message text.
#pragma once
#include <cstdint>
#include <memory>
#include <vector>

#include "parnn/data.hpp"
#include "parnn/error.hpp"
#include "parnn/network.hpp"
#include "parnn/parallel.hpp"
#include "parnn/pretrain.hpp"
#include "parnn_b200.h"

namespace parnn {
namespace b200 {

struct Options {
    int device = 0;
    int precision = PARNN_BF16;  // PARNN_FP32 for the fp32 parity mode
    // OptimizerKind::ngsgd runs the reference's kron-full NG-SGD by default; with
    // lowrank_ng it runs the online low-rank NG-SGD (rank-R Fisher projection and
    // subspace update; alpha = opts.ng_smoothing). 0 = the defaults (20, 80, 4, 2000, 3).
    bool lowrank_ng = false;
    int ng_rank_in = 0, ng_rank_out = 0, ng_update_period = 0, ng_update_lag = 0;
    double ng_history = 0.0;
};

namespace detail {
inline void check(int rc) {
    if (rc != PARNN_OK) fail(parnn_last_error());
}

class Ctx {
public:
    explicit Ctx(int dev) { check(parnn_ctx_create(dev, &c_)); }
    ~Ctx() { parnn_ctx_destroy(c_); }
    parnn_ctx* get() const { return c_; }

private:
    parnn_ctx* c_ = nullptr;
};

class Data {
public:
    Data(parnn_ctx* c, const Dataset& d) {
        std::vector<int32_t> y(d.labels.begin(), d.labels.end());
        check(parnn_dataset_create(c, d.features.data().data(), y.data(), d.size(), d.dim(), d.num_classes, &d_));
    }
    ~Data() { parnn_dataset_destroy(d_); }
    parnn_dataset* get() const { return d_; }

private:
    parnn_dataset* d_ = nullptr;
};

inline TrainResult run(const ParallelPlan& plan, const MlpModel& model0, const Dataset& train, const Dataset& cv,
                       const TrainOptions& opts, bool serial, const Options& o) {
    Ctx ctx(o.device);
    Data tr(ctx.get(), train);
    // The reference raises "train_parallel: empty CV set" itself for an empty cv.
    std::unique_ptr<Data> cvd;
    if (cv.size() > 0) cvd.reset(new Data(ctx.get(), cv));
    parnn_train_config cfg{};
    cfg.workers = plan.workers;
    cfg.avg_frequency = plan.avg_frequency;
    cfg.minibatch = plan.minibatch;
    cfg.base_seed = plan.base_seed;
    cfg.optimizer = opts.optimizer != OptimizerKind::ngsgd ? PARNN_SGD
                    : (o.lowrank_ng ? PARNN_NGSGD_LOWRANK : PARNN_NGSGD);
    cfg.ng_rank_in = o.ng_rank_in;
    cfg.ng_rank_out = o.ng_rank_out;
    cfg.ng_update_period = o.ng_update_period;
    cfg.ng_history = o.ng_history;
    cfg.ng_update_lag = o.ng_update_lag;
    cfg.lr_schedule = opts.lr_schedule == LrVariant::newbob ? PARNN_NEWBOB : PARNN_EXPONENTIAL;
    cfg.lr_init = opts.lr_init;
    cfg.epochs = opts.epochs;
    cfg.ng_decay = opts.ng_decay;
    cfg.ng_smoothing = opts.ng_smoothing;
    cfg.precision = o.precision;
    cfg.activation = model0.activation == Activation::sigmoid ? PARNN_SIGMOID : PARNN_TANH;
    cfg.serial = serial ? 1 : 0;
    std::vector<uint64_t> dims(model0.layer_dims.begin(), model0.layer_dims.end());
    const ParamVector p0 = flatten(model0);
    ParamVector p1;
    p1.data.resize(p0.size());
    std::vector<double> met(7 * (opts.epochs ? opts.epochs : 1));
    uint64_t ran = 0;
    check(parnn_train(ctx.get(), nullptr, &cfg, dims.data(), static_cast<int>(dims.size()), p0.data.data(), tr.get(),
                      cvd ? cvd->get() : nullptr, p1.data.data(), met.data(), &ran));
    TrainResult r;
    r.model = unflatten(p1, model0);
    for (uint64_t e = 0; e < ran; ++e) {
        const double* m = met.data() + 7 * e;
        EpochMetrics em;
        em.epoch = static_cast<std::size_t>(m[0]);
        em.lr = m[1];
        em.train_ce = m[2];
        em.cv_accuracy = m[3];
        em.wall_seconds = m[4];
        em.workers = static_cast<std::size_t>(m[5]);
        em.avg_events = static_cast<std::size_t>(m[6]);
        r.total_wall_seconds += em.wall_seconds;
        r.metrics.push_back(em);
    }
    return r;
}
}  // namespace detail

// parallel.hpp:73-75
inline TrainResult train_parallel(const ParallelPlan& plan, const MlpModel& model0, const Dataset& train,
                                  const Dataset& cv, const TrainOptions& opts, const Options& o = {}) {
    return detail::run(plan, model0, train, cv, opts, false, o);
}

// parallel.hpp:79-81
inline TrainResult serial_train(const MlpModel& model0, const Dataset& train, const Dataset& cv,
                                const TrainOptions& opts, std::size_t minibatch, std::uint64_t base_seed,
                                const Options& o = {}) {
    ParallelPlan p;
    p.workers = 1;
    p.avg_frequency = 1;
    p.minibatch = minibatch;
    p.base_seed = base_seed;
    return detail::run(p, model0, train, cv, opts, true, o);
}

}  // namespace b200
}  // namespace parnn
