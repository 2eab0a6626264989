// TEST INFRASTRUCTURE ONLY — C-ABI shim over the UNMODIFIED reference
// (/root/reference/proj/src/*.cpp, namespace parnn). Compiled by
// oracle/Makefile into oracle/_ref/libparnn_ref.so. Only tests/, the
// smoke check in __graft_entry__.py and bench.py's reference/cpu_baseline
// legs may load it; the product path never does.
//
// Every entry point takes/returns plain pointers (flatten order for model
// parameters, row-major doubles for matrices) and returns 0 on success or
// -1 after storing the reference's exception text (ref_last_error).
#include <algorithm>
#include <array>
#include <atomic>
#include <functional>
#include <mutex>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "parnn/data.hpp"
#include "parnn/error.hpp"
#include "parnn/network.hpp"
#include "parnn/optimizer.hpp"
#include "parnn/parallel.hpp"
#include "parnn/pretrain.hpp"
#include "parnn/rng.hpp"

using namespace parnn;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

std::vector<std::size_t> to_dims(const uint64_t* dims, int nd) {
    return std::vector<std::size_t>(dims, dims + nd);
}

MlpModel make_model(const uint64_t* dims, int nd, int act, const double* params) {
    MlpModel shape;
    shape.layer_dims = to_dims(dims, nd);
    shape.activation = act == 0 ? Activation::sigmoid : Activation::tanh;
    ParamVector pv;
    pv.data.assign(params, params + param_count(shape.layer_dims));
    return unflatten(pv, shape);
}

void put_params(const MlpModel& m, double* out) {
    const ParamVector pv = flatten(m);
    std::memcpy(out, pv.data.data(), pv.data.size() * sizeof(double));
}

Matrix make_matrix(const double* x, uint64_t r, uint64_t c) {
    return Matrix(r, c, std::vector<double>(x, x + r * c));
}

Dataset make_dataset(const double* x, const int32_t* y, uint64_t n, uint64_t d,
                     uint64_t classes) {
    Dataset ds;
    ds.features = make_matrix(x, n, d);
    ds.labels.assign(y, y + n);
    ds.num_classes = classes;
    return ds;
}

void put_grads(const GradientSet& g, double* out) {
    std::size_t pos = 0;
    for (const auto& l : g.layers) {
        std::memcpy(out + pos, l.weights.data().data(), l.weights.size() * sizeof(double));
        pos += l.weights.size();
        std::memcpy(out + pos, l.bias.data(), l.bias.size() * sizeof(double));
        pos += l.bias.size();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_param_count(const uint64_t* dims, int nd) {
    return param_count(to_dims(dims, nd));
}

// Raw xoshiro256** stream (rng.cpp:30-41) after splitmix64 seeding.
int ref_rng_u64(uint64_t seed, uint64_t n, uint64_t* out) {
    return guarded([&] {
        Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
    });
}

int ref_rng_uniform(uint64_t seed, uint64_t n, double* out) {
    return guarded([&] {
        Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
    });
}

int ref_rng_index(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out) {
    return guarded([&] {
        Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform_index(bound);
    });
}

int ref_rng_gaussian(uint64_t seed, uint64_t n, double mean, double stddev, double* out) {
    return guarded([&] {
        Rng r(seed);
        const auto v = r.gaussian_vector(n, mean, stddev);
        std::memcpy(out, v.data(), n * sizeof(double));
    });
}

int ref_shuffled_indices(uint64_t n, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        const auto v = shuffled_indices(n, seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = v[i];
    });
}

// Dataset generation + CV split + standardization exactly as BASELINE.md §4.3.
// Outputs: train (n_train x d) / cv (n_cv x d) features and labels.
int ref_make_data(uint64_t classes, uint64_t dim, uint64_t per_class, double sep,
                  uint64_t seed, double cv_fraction, uint64_t split_seed, int standardize,
                  double* train_x, int32_t* train_y, uint64_t* n_train, double* cv_x,
                  int32_t* cv_y, uint64_t* n_cv) {
    return guarded([&] {
        Dataset all = generate_synthetic(classes, dim, per_class, sep, seed);
        SplitSpec spec;
        spec.cv_fraction = cv_fraction;
        spec.seed = split_seed;
        auto [tr, cv] = split_cv(all, spec);
        if (standardize) {
            const FeatureStats st = feature_stats(tr);
            standardize_in_place(tr, st);
            standardize_in_place(cv, st);
        }
        *n_train = tr.size();
        *n_cv = cv.size();
        if (train_x) {
            std::memcpy(train_x, tr.features.data().data(), tr.features.size() * sizeof(double));
            for (std::size_t i = 0; i < tr.size(); ++i) train_y[i] = tr.labels[i];
        }
        if (cv_x) {
            std::memcpy(cv_x, cv.features.data().data(), cv.features.size() * sizeof(double));
            for (std::size_t i = 0; i < cv.size(); ++i) cv_y[i] = cv.labels[i];
        }
    });
}

int ref_generate_synthetic(uint64_t classes, uint64_t dim, uint64_t per_class, double sep,
                           uint64_t seed, double* x, int32_t* y) {
    return guarded([&] {
        Dataset ds = generate_synthetic(classes, dim, per_class, sep, seed);
        std::memcpy(x, ds.features.data().data(), ds.features.size() * sizeof(double));
        for (std::size_t i = 0; i < ds.size(); ++i) y[i] = ds.labels[i];
    });
}

int ref_feature_stats(const double* x, uint64_t n, uint64_t d, double* mean, double* stddev) {
    return guarded([&] {
        Dataset ds;
        ds.features = make_matrix(x, n, d);
        ds.labels.assign(n, 0);
        ds.num_classes = 1;
        const FeatureStats st = feature_stats(ds);
        std::memcpy(mean, st.mean.data(), d * sizeof(double));
        std::memcpy(stddev, st.stddev.data(), d * sizeof(double));
    });
}

// partition_data (parallel.cpp:61-77): returns, per shard, the row ids of the
// input dataset it holds (m * floor(N/m) entries, shard-major). Row identity is
// recovered by storing the row id as the single feature.
int ref_partition_rows(uint64_t n, uint64_t m, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        Dataset ds;
        ds.features = Matrix(n, 1);
        for (uint64_t i = 0; i < n; ++i) ds.features(i, 0) = static_cast<double>(i);
        ds.labels.assign(n, 0);
        ds.num_classes = 1;
        const auto shards = partition_data(ds, m, seed);
        std::size_t pos = 0;
        for (const auto& s : shards)
            for (std::size_t i = 0; i < s.size(); ++i) out[pos++] = static_cast<uint64_t>(s.features(i, 0));
    });
}

// minibatches (data.cpp:185-203) over a shard of n rows: the row order of
// all floor(n/B) batches concatenated.
int ref_minibatch_rows(uint64_t n, uint64_t batch, uint64_t epoch_seed, uint64_t* out) {
    return guarded([&] {
        Dataset ds;
        ds.features = Matrix(n, 1);
        for (uint64_t i = 0; i < n; ++i) ds.features(i, 0) = static_cast<double>(i);
        ds.labels.assign(n, 0);
        ds.num_classes = 1;
        const auto mbs = minibatches(ds, batch, epoch_seed);
        std::size_t pos = 0;
        for (const auto& mb : mbs)
            for (std::size_t i = 0; i < mb.features.rows(); ++i)
                out[pos++] = static_cast<uint64_t>(mb.features(i, 0));
    });
}

int ref_init_random(const uint64_t* dims, int nd, int act, uint64_t seed, double* params) {
    return guarded([&] {
        Rng rng(seed);
        const MlpModel m = init_random(to_dims(dims, nd), act == 0 ? Activation::sigmoid
                                                                    : Activation::tanh, rng);
        put_params(m, params);
    });
}

// forward (network.cpp:119-143) + cross_entropy (:145-160). z_out/a_out hold
// the concatenation over layers of B x d_{l+1} row-major blocks.
int ref_forward(const uint64_t* dims, int nd, int act, const double* params, const double* x,
                uint64_t batch, const int32_t* labels, double* z_out, double* a_out,
                double* ce_out) {
    return guarded([&] {
        const MlpModel m = make_model(dims, nd, act, params);
        const ForwardTrace tr = forward(m, make_matrix(x, batch, dims[0]));
        std::size_t pos = 0;
        for (std::size_t l = 0; l < tr.activations.size(); ++l) {
            const std::size_t sz = tr.activations[l].size();
            if (z_out) std::memcpy(z_out + pos, tr.pre_activations[l].data().data(), sz * sizeof(double));
            if (a_out) std::memcpy(a_out + pos, tr.activations[l].data().data(), sz * sizeof(double));
            pos += sz;
        }
        if (ce_out) *ce_out = cross_entropy(tr, Labels(labels, labels + batch));
    });
}

// backward_with_context (network.cpp:164-236): grads in flatten order,
// dz per layer concatenated (B x d_{l+1}).
int ref_backward(const uint64_t* dims, int nd, int act, const double* params, const double* x,
                 uint64_t batch, const int32_t* labels, double* grads, double* dz_out) {
    return guarded([&] {
        const MlpModel m = make_model(dims, nd, act, params);
        const ForwardTrace tr = forward(m, make_matrix(x, batch, dims[0]));
        BackpropContext ctx;
        const GradientSet g = backward_with_context(m, tr, Labels(labels, labels + batch), ctx);
        put_grads(g, grads);
        if (dz_out) {
            std::size_t pos = 0;
            for (const auto& d : ctx.dz) {
                std::memcpy(dz_out + pos, d.data().data(), d.size() * sizeof(double));
                pos += d.size();
            }
        }
    });
}

// One-replica training on explicit batches: for each of `steps` batches
// (rows of x given by row ids), forward -> CE -> backward -> [NG] -> SGD,
// exactly worker_epoch's body (parallel.cpp:117-130). lrs per step.
// Returns final params, per-step CE, and (if ng) the final NG factors
// concatenated as [r_in(l), r_out(l)] per layer, plus the last
// preconditioned gradient in flatten order.
int ref_train_steps(const uint64_t* dims, int nd, int act, const double* params0,
                    const double* x, uint64_t n_rows, const int32_t* labels,
                    const uint64_t* rows, uint64_t batch, uint64_t steps, const double* lrs,
                    int ngsgd, double ng_decay, double ng_smoothing, double* params_out,
                    double* ce_out, double* ng_factors_out, double* last_grad_out) {
    return guarded([&] {
        MlpModel m = make_model(dims, nd, act, params0);
        Dataset ds = make_dataset(x, labels, n_rows, dims[0], dims[nd - 1]);
        NgState ng = ng_init(m, ng_decay, ng_smoothing);
        for (uint64_t s = 0; s < steps; ++s) {
            const std::vector<std::size_t> sel(rows + s * batch, rows + (s + 1) * batch);
            const Dataset mb = ds.select(sel);
            const ForwardTrace tr = forward(m, mb.features);
            ce_out[s] = cross_entropy(tr, mb.labels);
            GradientSet g;
            if (ngsgd) {
                BackpropContext ctx;
                g = backward_with_context(m, tr, mb.labels, ctx);
                ng_update_state(ng, tr, ctx);
                g = ng_precondition(ng, g);
            } else {
                g = backward(m, tr, mb.labels);
            }
            if (last_grad_out && s + 1 == steps) put_grads(g, last_grad_out);
            sgd_step_in_place(m, g, lrs[s]);
        }
        put_params(m, params_out);
        if (ngsgd && ng_factors_out) {
            std::size_t pos = 0;
            for (const auto& l : ng.layers) {
                std::memcpy(ng_factors_out + pos, l.r_in.data().data(), l.r_in.size() * sizeof(double));
                pos += l.r_in.size();
                std::memcpy(ng_factors_out + pos, l.r_out.data().data(), l.r_out.size() * sizeof(double));
                pos += l.r_out.size();
            }
        }
    });
}

// ng_precondition on a single layer given explicit factors (optimizer.cpp:123-157).
int ref_ng_precondition_layer(uint64_t d_out, uint64_t d_in, const double* r_in,
                              const double* r_out, double smoothing, const double* gw,
                              const double* gb, double* out_w, double* out_b) {
    return guarded([&] {
        NgState st;
        st.smoothing = smoothing;
        NgLayerState ls;
        ls.r_in = make_matrix(r_in, d_in, d_in);
        ls.r_out = make_matrix(r_out, d_out, d_out);
        ls.update_count = 1;
        st.layers.push_back(ls);
        GradientSet g;
        g.layers.resize(1);
        g.layers[0].weights = make_matrix(gw, d_out, d_in);
        g.layers[0].bias.assign(gb, gb + d_out);
        const GradientSet o = ng_precondition(st, g);
        std::memcpy(out_w, o.layers[0].weights.data().data(), d_out * d_in * sizeof(double));
        std::memcpy(out_b, o.layers[0].bias.data(), d_out * sizeof(double));
    });
}

int ref_allreduce_average(const double* contributions, uint64_t m, uint64_t len, double* out) {
    return guarded([&] {
        std::vector<ParamVector> c(m);
        for (uint64_t r = 0; r < m; ++r) c[r].data.assign(contributions + r * len, contributions + (r + 1) * len);
        const ParamVector avg = allreduce_average(c, m);
        std::memcpy(out, avg.data.data(), len * sizeof(double));
    });
}

// train_parallel (parallel.cpp:279-283) / serial_train (:285-294) on explicit
// train/cv sets. metrics_out: epochs x 7 doubles
// [epoch, lr, train_ce, cv_accuracy, wall_seconds, workers, avg_events];
// returns the number of epochs actually run in *epochs_run.
int ref_train_parallel(const uint64_t* dims, int nd, int act, const double* params0,
                       const double* tx, const int32_t* ty, uint64_t n_train, const double* cx,
                       const int32_t* cy, uint64_t n_cv, uint64_t workers, uint64_t avg_frequency,
                       uint64_t minibatch, uint64_t base_seed, int ngsgd, int newbob, double lr_init,
                       uint64_t epochs, double ng_decay, double ng_smoothing, int serial,
                       double* params_out, double* metrics_out, uint64_t* epochs_run) {
    return guarded([&] {
        const MlpModel m0 = make_model(dims, nd, act, params0);
        const Dataset tr = make_dataset(tx, ty, n_train, dims[0], dims[nd - 1]);
        const Dataset cv = make_dataset(cx, cy, n_cv, dims[0], dims[nd - 1]);
        TrainOptions o;
        o.optimizer = ngsgd ? OptimizerKind::ngsgd : OptimizerKind::sgd;
        o.lr_schedule = newbob ? LrVariant::newbob : LrVariant::exponential;
        o.lr_init = lr_init;
        o.epochs = epochs;
        o.ng_decay = ng_decay;
        o.ng_smoothing = ng_smoothing;
        TrainResult r;
        if (serial) {
            r = serial_train(m0, tr, cv, o, minibatch, base_seed);
        } else {
            ParallelPlan p;
            p.workers = workers;
            p.avg_frequency = avg_frequency;
            p.minibatch = minibatch;
            p.base_seed = base_seed;
            r = train_parallel(p, m0, tr, cv, o);
        }
        put_params(r.model, params_out);
        *epochs_run = r.metrics.size();
        for (std::size_t e = 0; e < r.metrics.size(); ++e) {
            const auto& mt = r.metrics[e];
            double* row = metrics_out + 7 * e;
            row[0] = static_cast<double>(mt.epoch);
            row[1] = mt.lr;
            row[2] = mt.train_ce;
            row[3] = mt.cv_accuracy;
            row[4] = mt.wall_seconds;
            row[5] = static_cast<double>(mt.workers);
            row[6] = static_cast<double>(mt.avg_events);
        }
    });
}

double ref_accuracy(const uint64_t* dims, int nd, int act, const double* params,
                    const double* x, uint64_t n, const int32_t* y) {
    double acc = -1.0;
    guarded([&] {
        const MlpModel m = make_model(dims, nd, act, params);
        acc = accuracy(m, make_matrix(x, n, dims[0]), Labels(y, y + n));
    });
    return acc;
}

// LR schedule primitives (optimizer.cpp:169-208).
int ref_newbob_sequence(double lr_init, const double* accs, uint64_t n, double* lr_out,
                        int* stop_out) {
    return guarded([&] {
        LrSchedule s = make_schedule(LrVariant::newbob, lr_init, 15);
        for (uint64_t i = 1; i < n; ++i) {
            const NewbobDecision d = newbob_next(s, accs[i - 1], accs[i]);
            lr_out[i - 1] = d.lr;
            stop_out[i - 1] = d.stop ? 1 : 0;
        }
    });
}

double ref_exponential_lr(double lr_init, uint64_t epochs, double progress) {
    double v = -1.0;
    guarded([&] { v = exponential_lr(make_schedule(LrVariant::exponential, lr_init, epochs), progress); });
    return v;
}

// RBM (pretrain.cpp). Parameters packed as [W (h x v), v_bias (v), h_bias (h)].
static RbmParams make_rbm(uint64_t v, uint64_t h, int gaussian, const double* p) {
    RbmParams r;
    r.weights = make_matrix(p, h, v);
    r.v_bias.assign(p + h * v, p + h * v + v);
    r.h_bias.assign(p + h * v + v, p + h * v + v + h);
    r.visible_kind = gaussian ? VisibleKind::gaussian : VisibleKind::bernoulli;
    return r;
}

static void put_rbm(const RbmParams& r, double* p) {
    const std::size_t hv = r.weights.size();
    std::memcpy(p, r.weights.data().data(), hv * sizeof(double));
    std::memcpy(p + hv, r.v_bias.data(), r.v_bias.size() * sizeof(double));
    std::memcpy(p + hv + r.v_bias.size(), r.h_bias.data(), r.h_bias.size() * sizeof(double));
}

int ref_rbm_init(uint64_t v, uint64_t h, int gaussian, uint64_t seed, double* p) {
    return guarded([&] {
        Rng rng(seed);
        put_rbm(rbm_init(v, h, gaussian ? VisibleKind::gaussian : VisibleKind::bernoulli, rng), p);
    });
}

// mode 0: rng sampling with Rng(seed); mode 1: threshold_half stub.
// trace_out (nullable): [pos_hidden, hidden_sample, recon, neg_hidden].
int ref_cd1_update(uint64_t v, uint64_t h, int gaussian, const double* p, const double* batch,
                   uint64_t b, double lr, int mode, uint64_t seed, double* p_out,
                   double* trace_out) {
    return guarded([&] {
        const RbmParams r = make_rbm(v, h, gaussian, p);
        const Matrix bm = make_matrix(batch, b, v);
        Cd1Trace tr;
        if (mode == 0) {
            Rng rng(seed);
            tr = cd1_gibbs(r, bm, rng);
        } else {
            tr.pos_hidden = hidden_probs(r, bm);
            tr.hidden_sample = threshold_half(tr.pos_hidden);
            tr.recon = reconstruct_mean(r, tr.hidden_sample);
            tr.neg_hidden = hidden_probs(r, tr.recon);
        }
        put_rbm(cd1_apply(r, bm, tr, lr), p_out);
        if (trace_out) {
            double* o = trace_out;
            for (const Matrix* mm : {&tr.pos_hidden, &tr.hidden_sample, &tr.recon, &tr.neg_hidden}) {
                std::memcpy(o, mm->data().data(), mm->size() * sizeof(double));
                o += mm->size();
            }
        }
    });
}

// cd1_apply on an explicit trace (pretrain.cpp:89-121).
int ref_cd1_apply(uint64_t v, uint64_t h, int gaussian, const double* p, const double* batch,
                  uint64_t b, const double* pos_h, const double* recon, const double* neg_h,
                  double lr, double* p_out) {
    return guarded([&] {
        const RbmParams r = make_rbm(v, h, gaussian, p);
        Cd1Trace tr;
        tr.pos_hidden = make_matrix(pos_h, b, h);
        tr.hidden_sample = tr.pos_hidden;
        tr.recon = make_matrix(recon, b, v);
        tr.neg_hidden = make_matrix(neg_h, b, h);
        put_rbm(cd1_apply(r, make_matrix(batch, b, v), tr, lr), p_out);
    });
}

double ref_reconstruction_error(uint64_t v, uint64_t h, int gaussian, const double* p,
                                const double* batch, uint64_t b) {
    double e = -1.0;
    guarded([&] { e = reconstruction_error(make_rbm(v, h, gaussian, p), make_matrix(batch, b, v)); });
    return e;
}

int ref_greedy_pretrain(const uint64_t* dims, int nd, const double* data, uint64_t n,
                        uint64_t epochs, double lr_g, double lr_b, uint64_t batch, uint64_t seed,
                        double* params_out) {
    return guarded([&] {
        PretrainOptions o;
        o.epochs = epochs;
        o.lr_gaussian = lr_g;
        o.lr_bernoulli = lr_b;
        o.batch_size = batch;
        Rng rng(seed);
        put_params(greedy_pretrain(to_dims(dims, nd), make_matrix(data, n, dims[0]), o,
                                   Activation::sigmoid, rng),
                   params_out);
    });
}

int ref_save_model(const char* path, const uint64_t* dims, int nd, int act, const double* params) {
    return guarded([&] { save_model(path, make_model(dims, nd, act, params)); });
}

// Reads a PARNNET1 file; *nd in/out (capacity in, count out).
int ref_load_model(const char* path, uint64_t* dims, int* nd, int* act, double* params,
                   uint64_t cap) {
    return guarded([&] {
        const MlpModel m = load_model(path);
        if (static_cast<std::size_t>(*nd) < m.layer_dims.size()) fail("ref_load_model: dims capacity");
        *nd = static_cast<int>(m.layer_dims.size());
        for (std::size_t i = 0; i < m.layer_dims.size(); ++i) dims[i] = m.layer_dims[i];
        *act = m.activation == Activation::sigmoid ? 0 : 1;
        const ParamVector pv = flatten(m);
        if (pv.size() > cap) fail("ref_load_model: params capacity");
        std::memcpy(params, pv.data.data(), pv.size() * sizeof(double));
    });
}

// ---- CPU-baseline timing (bench.py --impl reference / cpu_baseline) -------
// Times the reference's own per-minibatch path (parallel.cpp:117-130) on
// `threads` concurrent workers, each a private replica on its own batch
// stream, for `steps` steps. Returns total frames processed / wall seconds
// and the per-phase seconds of worker 0 in phase_out[5] =
// {forward+ce, backward, ng_update_state, ng_precondition, sgd}.
double ref_time_steps(const uint64_t* dims, int nd, const double* params0, const double* x,
                      uint64_t n_rows, const int32_t* labels, uint64_t batch, uint64_t steps,
                      int ngsgd, int threads, double* phase_out) {
    double fps = -1.0;
    guarded([&] {
        const MlpModel m0 = make_model(dims, nd, 0, params0);
        const Dataset ds = make_dataset(x, labels, n_rows, dims[0], dims[nd - 1]);
        std::vector<std::array<double, 5>> phases(threads);
        auto work = [&](int t) {
            MlpModel m = m0;
            NgState ng = ng_init(m);
            Rng rng(1000 + t);
            auto& ph = phases[t];
            ph.fill(0.0);
            for (uint64_t s = 0; s < steps; ++s) {
                std::vector<std::size_t> sel(batch);
                for (auto& r : sel) r = rng.uniform_index(n_rows);
                const Dataset mb = ds.select(sel);
                auto t0 = std::chrono::steady_clock::now();
                const ForwardTrace tr = forward(m, mb.features);
                volatile double ce = cross_entropy(tr, mb.labels);
                (void)ce;
                auto t1 = std::chrono::steady_clock::now();
                GradientSet g;
                BackpropContext ctx;
                if (ngsgd) g = backward_with_context(m, tr, mb.labels, ctx);
                else g = backward(m, tr, mb.labels);
                auto t2 = std::chrono::steady_clock::now();
                if (ngsgd) ng_update_state(ng, tr, ctx);
                auto t3 = std::chrono::steady_clock::now();
                if (ngsgd) g = ng_precondition(ng, g);
                auto t4 = std::chrono::steady_clock::now();
                sgd_step_in_place(m, g, 1e-6);
                auto t5 = std::chrono::steady_clock::now();
                ph[0] += std::chrono::duration<double>(t1 - t0).count();
                ph[1] += std::chrono::duration<double>(t2 - t1).count();
                ph[2] += std::chrono::duration<double>(t3 - t2).count();
                ph[3] += std::chrono::duration<double>(t4 - t3).count();
                ph[4] += std::chrono::duration<double>(t5 - t4).count();
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
        for (auto& t : th) t.join();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fps = static_cast<double>(threads) * static_cast<double>(steps * batch) / wall;
        if (phase_out)
            for (int i = 0; i < 5; ++i) phase_out[i] = phases[0][i];
    });
    return fps;
}

// ---- One TRUE-WIDTH minibatch step of the reference on all host cores -----
// worker_epoch's body for one minibatch (parallel.cpp:117-130) -- forward,
// cross_entropy, backward_with_context, ng_update_state, ng_precondition,
// sgd_step_in_place -- built only from the reference's own public functions
// (forward, cross_entropy, backward_with_context, matmul_tn, smoothed_factor,
// cholesky_solve, transpose, frobenius_norm, sgd_step_in_place), spread over
// `threads` host threads along the only seams those functions allow without
// changing their arithmetic:
//   * forward / cross_entropy / backward_with_context on row chunks of the
//     batch (every output row and every dz row is computed exactly as in the
//     whole-batch call); the per-chunk gradients dz_c^T A_c / b_c are combined
//     as sum_c (b_c / B) g_c  (the whole-batch call sums all rows, then / B);
//   * the NG moments A^T A / B, D^T D / B as per-chunk matmul_tn partials,
//     summed (ng_update_state, optimizer.cpp:79-106; first update: r = C);
//   * ng_precondition (optimizer.cpp:123-157) with its two cholesky_solve calls
//     split over right-hand-side columns (each task refactors S, exactly as
//     every reference call does), the bias solve (a further S_out factor) as
//     its own task, gamma from the full Frobenius norms.
// Tasks of a phase run longest-first on a dynamic pool. The result equals the
// single-threaded reference step up to fp64 summation order (checked by
// tests/test_oracle.py at a small shape against ref_train_steps).
// phase_out[7] = seconds of {forward+ce, backward (+combine), moments,
// smoothed factors + first solves + bias solves, second solves, gamma +
// assemble, sgd}; returns the step's wall seconds (or -1 on error).
double ref_time_step_threaded(const uint64_t* dims, int nd, const double* params0, const double* x,
                              const int32_t* labels, uint64_t batch, int ngsgd, int threads, double lr,
                              double* phase_out, double* params_out, double* ce_out) {
    double wall = -1.0;
    guarded([&] {
        using clk = std::chrono::steady_clock;
        const int T = std::max(1, threads);
        MlpModel m = make_model(dims, nd, 0, params0);
        const std::size_t L = m.layers.size();
        const Matrix X = make_matrix(x, batch, dims[0]);
        const Labels Y(labels, labels + batch);
        auto pool = [&](std::vector<std::pair<double, std::function<void()>>>& tasks) {
            std::sort(tasks.begin(), tasks.end(), [](auto& a, auto& b) { return a.first > b.first; });
            std::atomic<std::size_t> next{0};
            std::vector<std::thread> th;
            std::mutex emu;
            std::string err;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&] {
                    for (std::size_t i; (i = next.fetch_add(1)) < tasks.size();) {
                        try {
                            tasks[i].second();
                        } catch (const std::exception& e) {
                            std::lock_guard<std::mutex> lk(emu);
                            err = e.what();
                        }
                    }
                });
            for (auto& t : th) t.join();
            if (!err.empty()) throw std::runtime_error(err);
        };
        // row chunks of the batch
        const std::size_t nch = std::min<std::size_t>(T, batch);
        std::vector<std::size_t> r0(nch + 1);
        for (std::size_t c = 0; c <= nch; ++c) r0[c] = batch * c / nch;
        std::vector<Matrix> xc(nch);
        std::vector<Labels> yc(nch);
        for (std::size_t c = 0; c < nch; ++c) {
            const std::size_t b = r0[c + 1] - r0[c];
            xc[c] = Matrix(b, dims[0], std::vector<double>(X.row_ptr(r0[c]), X.row_ptr(r0[c]) + b * dims[0]));
            yc[c].assign(Y.begin() + r0[c], Y.begin() + r0[c + 1]);
        }
        std::vector<ForwardTrace> trc(nch);
        std::vector<double> cec(nch);
        std::vector<GradientSet> gc(nch);
        std::vector<BackpropContext> cxc(nch);
        std::vector<std::pair<double, std::function<void()>>> tasks;
        double ph[7] = {0, 0, 0, 0, 0, 0, 0};
        const auto t_all = clk::now();
        auto tick = clk::now();
        auto lap = [&](int i) {
            const auto now = clk::now();
            ph[i] = std::chrono::duration<double>(now - tick).count();
            tick = now;
        };
        // forward + cross_entropy
        for (std::size_t c = 0; c < nch; ++c)
            tasks.push_back({1.0, [&, c] {
                                 trc[c] = forward(m, xc[c]);
                                 cec[c] = cross_entropy(trc[c], yc[c]);
                             }});
        pool(tasks);
        tasks.clear();
        double ce = 0.0;
        for (std::size_t c = 0; c < nch; ++c) ce += cec[c] * static_cast<double>(r0[c + 1] - r0[c]);
        ce /= static_cast<double>(batch);
        lap(0);
        // backward (+ combine sum_c (b_c / B) g_c, per layer)
        for (std::size_t c = 0; c < nch; ++c)
            tasks.push_back({1.0, [&, c] { gc[c] = backward_with_context(m, trc[c], yc[c], cxc[c]); }});
        pool(tasks);
        tasks.clear();
        GradientSet g;
        g.layers.resize(L);
        for (std::size_t l = 0; l < L; ++l)
            tasks.push_back({static_cast<double>(gc[0].layers[l].weights.size()), [&, l] {
                                 LayerParams& o = g.layers[l];
                                 o.weights = Matrix(gc[0].layers[l].weights.rows(), gc[0].layers[l].weights.cols());
                                 o.bias.assign(gc[0].layers[l].bias.size(), 0.0);
                                 for (std::size_t c = 0; c < nch; ++c) {
                                     const double f = static_cast<double>(r0[c + 1] - r0[c]) / static_cast<double>(batch);
                                     const auto& gw = gc[c].layers[l].weights.data();
                                     auto& ow = o.weights.data();
                                     for (std::size_t i = 0; i < ow.size(); ++i) ow[i] += f * gw[i];
                                     for (std::size_t i = 0; i < o.bias.size(); ++i) o.bias[i] += f * gc[c].layers[l].bias[i];
                                 }
                             }});
        pool(tasks);
        tasks.clear();
        lap(1);
        GradientSet out = g;
        if (ngsgd) {
            // moments: per (layer, side, chunk) matmul_tn partials, then sums x 1/B
            std::vector<std::vector<Matrix>> part(2 * L, std::vector<Matrix>(nch));
            for (std::size_t l = 0; l < L; ++l)
                for (int sd = 0; sd < 2; ++sd)
                    for (std::size_t c = 0; c < nch; ++c)
                        tasks.push_back({static_cast<double>(sd ? dims[l + 1] * dims[l + 1] : dims[l] * dims[l]),
                                         [&, l, sd, c] {
                                             const Matrix& a = sd ? cxc[c].dz[l]
                                                                  : (l == 0 ? trc[c].input : trc[c].activations[l - 1]);
                                             part[2 * l + sd][c] = matmul_tn(a, a);
                                         }});
            pool(tasks);
            tasks.clear();
            std::vector<Matrix> rfac(2 * L);
            for (std::size_t i = 0; i < 2 * L; ++i)
                tasks.push_back({static_cast<double>(part[i][0].size()), [&, i] {
                                     Matrix s = part[i][0];
                                     for (std::size_t c = 1; c < nch; ++c) {
                                         auto& d = s.data();
                                         const auto& p = part[i][c].data();
                                         for (std::size_t k = 0; k < d.size(); ++k) d[k] += p[k];
                                     }
                                     scale_in_place(s, 1.0 / static_cast<double>(batch));
                                     rfac[i] = std::move(s);  // ema_update, t = 1: r = C
                                     part[i].clear();
                                 }});
            pool(tasks);
            tasks.clear();
            lap(2);
            // smoothed factors, then the first solves S_out^-1 G (column chunks) and the bias solves
            std::vector<Matrix> sfac(2 * L);
            for (std::size_t i = 0; i < 2 * L; ++i)
                tasks.push_back({static_cast<double>(rfac[i].size()), [&, i] { sfac[i] = smoothed_factor(rfac[i], 4.0); }});
            pool(tasks);
            tasks.clear();
            auto col_chunks = [&](std::size_t nrow, std::size_t ncol) {
                // a factor that costs more than the solves (output layer: 8806 rows vs 2048 columns)
                // is refactored by every chunk: T - 1 chunks, one thread left for the bias solve
                std::size_t k = nrow > 2 * ncol ? static_cast<std::size_t>(std::max(1, T - 1)) : 4;
                return std::max<std::size_t>(1, std::min<std::size_t>(k, ncol / 32));
            };
            auto cols_of = [](const Matrix& a, std::size_t c0, std::size_t c1) {
                Matrix o(a.rows(), c1 - c0);
                for (std::size_t r = 0; r < a.rows(); ++r)
                    std::copy(a.row_ptr(r) + c0, a.row_ptr(r) + c1, o.row_ptr(r));
                return o;
            };
            std::vector<std::vector<Matrix>> left(L), right(L);
            std::vector<Matrix> bhat(L);
            std::vector<std::vector<std::size_t>> cb1(L), cb2(L);
            for (std::size_t l = 0; l < L; ++l) {
                const Matrix& G = g.layers[l].weights;  // dout x din
                const double n_out = static_cast<double>(dims[l + 1]);
                const std::size_t k1 = col_chunks(dims[l + 1], G.cols());
                left[l].resize(k1);
                for (std::size_t c = 0; c <= k1; ++c) cb1[l].push_back(G.cols() * c / k1);
                for (std::size_t c = 0; c < k1; ++c)
                    tasks.push_back({n_out * n_out * n_out / 3.0 + 2.0 * n_out * n_out * (cb1[l][c + 1] - cb1[l][c]),
                                     [&, l, c] {
                                         left[l][c] = cholesky_solve(sfac[2 * l + 1], cols_of(g.layers[l].weights,
                                                                                              cb1[l][c], cb1[l][c + 1]));
                                     }});
                tasks.push_back({n_out * n_out * n_out / 3.0, [&, l] {
                                     Matrix bias_col(g.layers[l].bias.size(), 1, g.layers[l].bias);
                                     bhat[l] = cholesky_solve(sfac[2 * l + 1], bias_col);
                                 }});
            }
            pool(tasks);
            tasks.clear();
            lap(3);
            // second solves S_in^-1 (S_out^-1 G)^T over column chunks of the transpose
            std::vector<Matrix> leftT(L);
            for (std::size_t l = 0; l < L; ++l) {
                Matrix lf(g.layers[l].weights.rows(), g.layers[l].weights.cols());
                for (std::size_t c = 0; c < left[l].size(); ++c)
                    for (std::size_t r = 0; r < lf.rows(); ++r)
                        std::copy(left[l][c].row_ptr(r), left[l][c].row_ptr(r) + left[l][c].cols(),
                                  lf.row_ptr(r) + cb1[l][c]);
                leftT[l] = transpose(lf);  // din x dout
                const double n_in = static_cast<double>(dims[l]);
                const std::size_t k2 = std::min<std::size_t>(static_cast<std::size_t>(T),
                                                             std::max<std::size_t>(1, leftT[l].cols() / 512));
                right[l].resize(k2);
                for (std::size_t c = 0; c <= k2; ++c) cb2[l].push_back(leftT[l].cols() * c / k2);
                for (std::size_t c = 0; c < k2; ++c)
                    tasks.push_back({n_in * n_in * n_in / 3.0 + 2.0 * n_in * n_in * (cb2[l][c + 1] - cb2[l][c]),
                                     [&, l, c] {
                                         right[l][c] = cholesky_solve(sfac[2 * l], cols_of(leftT[l], cb2[l][c], cb2[l][c + 1]));
                                     }});
            }
            pool(tasks);
            tasks.clear();
            lap(4);
            // assemble ghat = transpose(S_in^-1 left^T), gamma rescales (optimizer.cpp:141-154)
            for (std::size_t l = 0; l < L; ++l)
                tasks.push_back({static_cast<double>(g.layers[l].weights.size()), [&, l] {
                                     Matrix rt(leftT[l].rows(), leftT[l].cols());
                                     for (std::size_t c = 0; c < right[l].size(); ++c)
                                         for (std::size_t r = 0; r < rt.rows(); ++r)
                                             std::copy(right[l][c].row_ptr(r), right[l][c].row_ptr(r) + right[l][c].cols(),
                                                       rt.row_ptr(r) + cb2[l][c]);
                                     Matrix ghat = transpose(rt);
                                     const double gamma = frobenius_norm(g.layers[l].weights) /
                                                          std::max(frobenius_norm(ghat), 1e-20);
                                     scale_in_place(ghat, gamma);
                                     out.layers[l].weights = std::move(ghat);
                                     const double gamma_b = frobenius_norm(g.layers[l].bias) /
                                                            std::max(frobenius_norm(bhat[l]), 1e-20);
                                     for (std::size_t i = 0; i < g.layers[l].bias.size(); ++i)
                                         out.layers[l].bias[i] = gamma_b * bhat[l](i, 0);
                                 }});
            pool(tasks);
            tasks.clear();
            lap(5);
        }
        sgd_step_in_place(m, out, lr);
        lap(6);
        wall = std::chrono::duration<double>(clk::now() - t_all).count();
        if (phase_out)
            for (int i = 0; i < 7; ++i) phase_out[i] = ph[i];
        if (params_out) put_params(m, params_out);
        if (ce_out) *ce_out = ce;
    });
    return wall;
}

// Times ng_precondition alone for one layer shape (d_out x d_in) with
// factors built from `batch` random rows; returns seconds per call.
double ref_time_ng_precondition(uint64_t d_out, uint64_t d_in, uint64_t batch, uint64_t seed) {
    double secs = -1.0;
    guarded([&] {
        Rng rng(seed);
        MlpModel m;
        m.layer_dims = {d_in, d_out};
        m.activation = Activation::sigmoid;
        LayerParams p;
        p.weights = Matrix(d_out, d_in);
        for (double& w : p.weights.data()) w = rng.uniform(-0.1, 0.1);
        p.bias.assign(d_out, 0.0);
        m.layers.push_back(p);
        NgState ng = ng_init(m);
        ng.layers[0].r_in = Matrix(d_in, d_in);
        ng.layers[0].r_out = Matrix(d_out, d_out);
        Matrix a(batch, d_in), d(batch, d_out);
        for (double& v : a.data()) v = rng.uniform();
        for (double& v : d.data()) v = rng.uniform(-0.01, 0.01);
        ng.layers[0].r_in = matmul_tn(a, a);
        ng.layers[0].r_out = matmul_tn(d, d);
        ng.layers[0].update_count = 1;
        GradientSet g;
        g.layers.resize(1);
        g.layers[0].weights = Matrix(d_out, d_in);
        for (double& v : g.layers[0].weights.data()) v = rng.uniform(-1e-3, 1e-3);
        g.layers[0].bias.assign(d_out, 1e-4);
        const auto t0 = std::chrono::steady_clock::now();
        const GradientSet o = ng_precondition(ng, g);
        secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        volatile double sink = o.layers[0].weights(0, 0);
        (void)sink;
    });
    return secs;
}

}  // extern "C"

// load_csv / save_csv (data.cpp:66-122) of the reference, for the CSV parity tests.
extern "C" int ref_load_csv(const char* path, double* x, int32_t* y, uint64_t cap_rows, uint64_t cap_dim,
                            uint64_t* n, uint64_t* d, uint64_t* classes) {
    return guarded([&] {
        const Dataset ds = load_csv(path);
        *n = ds.size();
        *d = ds.dim();
        *classes = ds.num_classes;
        if (x && y && ds.size() <= cap_rows && ds.dim() <= cap_dim) {
            std::memcpy(x, ds.features.data().data(), ds.features.size() * sizeof(double));
            for (std::size_t i = 0; i < ds.size(); ++i) y[i] = ds.labels[i];
        }
    });
}

extern "C" int ref_save_csv(const char* path, const double* x, const int32_t* y, uint64_t n, uint64_t d) {
    return guarded([&] { save_csv(path, make_dataset(x, y, n, d, 1)); });
}
