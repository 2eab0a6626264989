// Reference-side adapter: the parnn C++ API (namespace parnn, reference
// headers parallel.hpp / network.hpp / pretrain.hpp) implemented on top of the
// B200 C ABI (include/parnn_b200.h). A maintainer of the reference swaps the
// body of parnn::train_parallel / serial_train / greedy_pretrain
// (parallel.cpp:279-294, pretrain.cpp:162-207) for these calls; every value
// type stays the reference's own, and errors come back as parnn::Error with
// the reference's message text.
#pragma once
#include <cstdint>
#include <cstring>
#include <memory>
#include <type_traits>
#include <vector>

#include "parnn/data.hpp"
#include "parnn/error.hpp"
#include "parnn/network.hpp"
#include "parnn/parallel.hpp"
#include "parnn/pretrain.hpp"
#include "parnn/rng.hpp"
#include "parnn_b200.h"

namespace parnn {
namespace b200 {

struct Options {
    int device = 0;
    // PARNN_FP32 (3xTF32 operands, fp32 everything else) is the default: the
    // closest to the reference's fp64 results. PARNN_BF16 is the fast mode.
    int precision = PARNN_FP32;
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

// pretrain.hpp:74-76. The caller's Rng is advanced exactly as the reference's
// greedy_pretrain advances it (rbm_init, the per-epoch shuffles, the Bernoulli
// draws it would consume, the output-layer init); its state crosses the C ABI
// as the object's own words. parnn::Rng is a standard-layout, trivially
// copyable class {uint64_t state_[4]; double spare_; bool has_spare_;}
// (rng.hpp), so its bytes are read and written with memcpy.
inline MlpModel greedy_pretrain(const std::vector<std::size_t>& dims, const Matrix& data,
                                const PretrainOptions& opts, Activation activation, Rng& rng,
                                const Options& o = {}) {
    static_assert(std::is_trivially_copyable_v<Rng> && std::is_standard_layout_v<Rng>, "Rng layout");
    static_assert(sizeof(Rng) == 48, "Rng = {uint64_t[4], double, bool}");
    if (dims.size() < 2) fail("greedy_pretrain: need at least 2 dims");
    if (data.cols() != dims.front())
        fail("greedy_pretrain: data has ", data.cols(), " columns, dims expect ", dims.front());
    if (opts.batch_size == 0) fail("greedy_pretrain: batch size must be >= 1");
    unsigned char raw[sizeof(Rng)];
    std::memcpy(raw, &rng, sizeof(Rng));
    uint64_t st[4];
    double spare = 0.0;
    bool has = false;
    std::memcpy(st, raw, 32);
    std::memcpy(&spare, raw + 32, 8);
    std::memcpy(&has, raw + 40, 1);
    int has_i = has ? 1 : 0;
    detail::Ctx ctx(o.device);
    std::vector<uint64_t> d(dims.begin(), dims.end());
    MlpModel shape;
    shape.layer_dims = dims;
    shape.activation = activation;
    ParamVector p;
    p.data.resize(param_count(dims));
    detail::check(parnn_greedy_pretrain_rng(ctx.get(), d.data(), static_cast<int>(d.size()), data.data().data(),
                                            data.rows(), opts.epochs, opts.lr_gaussian, opts.lr_bernoulli,
                                            opts.batch_size,
                                            activation == Activation::sigmoid ? PARNN_SIGMOID : PARNN_TANH, st,
                                            &spare, &has_i, o.precision, p.data.data()));
    std::memcpy(raw, st, 32);
    std::memcpy(raw + 32, &spare, 8);
    has = has_i != 0;
    std::memcpy(raw + 40, &has, 1);
    std::memcpy(static_cast<void*>(&rng), raw, sizeof(Rng));
    return unflatten(p, shape);
}

}  // namespace b200
}  // namespace parnn
