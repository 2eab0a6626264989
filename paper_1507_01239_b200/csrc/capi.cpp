// extern "C" boundary (include/parnn_b200.h). Never throws across the ABI:
// every entry point converts exceptions into PARNN_ERR + parnn_last_error().
#include "../../include/parnn_b200.h"

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "host.h"
#include "parallel.h"
#include "rbm.h"

using namespace pnb;

struct parnn_ctx {
    std::unique_ptr<Context> c;
};
struct parnn_dataset {
    std::unique_ptr<DeviceDataset> d;
};
struct parnn_replica {
    std::unique_ptr<Replica> r;
};
struct parnn_comm {
    std::unique_ptr<Comm> c;
};
struct parnn_rbm {
    std::unique_ptr<RbmDevice> r;
};
struct parnn_averager {
    std::unique_ptr<Averager> a;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return PARNN_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
    } catch (...) {
        g_err = "unknown error";
    }
    return PARNN_ERR;
}

void need(const void* p, const char* what) {
    if (!p) throw std::runtime_error(std::string(what) + ": null pointer");
}

std::vector<long> to_dims(const uint64_t* dims, int nd) {
    need(dims, "dims");
    if (nd < 2) throw std::runtime_error("init_random: need at least 2 dims, got " + std::to_string(nd));
    std::vector<long> v;
    for (int i = 0; i < nd; ++i) v.push_back(static_cast<long>(dims[i]));
    return v;
}

uint64_t padded_factor_count(const Replica& r) {
    uint64_t n = 0;
    for (int l = 0; l < r.L; ++l) n += r.dims[l] * r.dims[l] + r.dims[l + 1] * r.dims[l + 1];
    return n;
}

uint64_t flat_count(const Replica& r) {
    uint64_t n = 0;
    for (int l = 0; l < r.L; ++l) n += r.dims[l] * r.dims[l + 1] + r.dims[l + 1];
    return n;
}
}  // namespace

extern "C" {

const char* parnn_last_error(void) { return g_err.c_str(); }
const char* parnn_version(void) { return "parnn_b200 0.1 (sm_100a)"; }

int parnn_rng_u64(uint64_t seed, uint64_t n, uint64_t* out) {
    return guarded([&] {
        host::Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
    });
}

int parnn_rng_uniform(uint64_t seed, uint64_t n, double* out) {
    return guarded([&] {
        host::Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
    });
}

int parnn_rng_gaussian(uint64_t seed, uint64_t n, double mean, double stddev, double* out) {
    return guarded([&] {
        host::Rng r(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = r.gaussian(mean, stddev);
    });
}

int parnn_shuffled_indices(uint64_t n, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        const auto v = host::shuffled_indices(n, seed);
        std::memcpy(out, v.data(), n * 8);
    });
}

int parnn_partition_rows(uint64_t n, uint64_t m, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        const auto v = host::partition_rows(n, m, seed);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

int parnn_minibatch_rows(uint64_t n, uint64_t b, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        const auto v = host::minibatch_rows(n, b, seed);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

int parnn_make_data(uint64_t classes, uint64_t dim, uint64_t per_class, double sep, uint64_t seed, double cv_fraction,
                    uint64_t split_seed, int standardize, double* train_x, int32_t* train_y, uint64_t* n_train,
                    double* cv_x, int32_t* cv_y, uint64_t* n_cv) {
    return guarded([&] {
        const host::HostData all = host::generate_synthetic(classes, dim, per_class, sep, seed);
        host::HostData tr, cv;
        host::split_cv(all, cv_fraction, split_seed, tr, cv);
        if (standardize) {
            std::vector<double> mu, sd;
            host::feature_stats(tr, mu, sd);
            host::standardize(tr, mu, sd);
            host::standardize(cv, mu, sd);
        }
        *n_train = tr.n;
        *n_cv = cv.n;
        if (train_x) std::memcpy(train_x, tr.x.data(), tr.x.size() * 8);
        if (train_y) std::memcpy(train_y, tr.y.data(), tr.y.size() * 4);
        if (cv_x) std::memcpy(cv_x, cv.x.data(), cv.x.size() * 8);
        if (cv_y) std::memcpy(cv_y, cv.y.data(), cv.y.size() * 4);
    });
}

uint64_t parnn_param_count(const uint64_t* dims, int nd) {
    return host::param_count(std::vector<uint64_t>(dims, dims + nd));
}

int parnn_init_random(const uint64_t* dims, int nd, uint64_t seed, double* params) {
    return guarded([&] {
        host::Rng r(seed);
        const auto p = host::init_random(std::vector<uint64_t>(dims, dims + nd), r);
        std::memcpy(params, p.data(), p.size() * 8);
    });
}

int parnn_exponential_lr(double lr_init, uint64_t epochs, double progress, double* lr) {
    return guarded([&] { *lr = host::exponential_lr(host::make_schedule(false, lr_init, epochs), progress); });
}

int parnn_newbob_sequence(double lr_init, const double* accs, uint64_t n, double* lr_out, int* stop_out) {
    return guarded([&] {
        host::Schedule s = host::make_schedule(true, lr_init, 15);
        for (uint64_t i = 1; i < n; ++i) stop_out[i - 1] = host::newbob_next(s, accs[i - 1], accs[i], &lr_out[i - 1]);
    });
}

int parnn_scale_lr_for_workers(double lr_init, uint64_t workers, double* lr) {
    return guarded([&] { *lr = host::scale_lr_for_workers(lr_init, workers); });
}

int parnn_save_model(const char* path, const uint64_t* dims, int nd, int act, const double* params) {
    return guarded([&] {
        std::vector<uint64_t> d(dims, dims + nd);
        host::save_model(path, d, act, std::vector<double>(params, params + host::param_count(d)));
    });
}

int parnn_load_model(const char* path, uint64_t* dims, int* nd, int* act, double* params, uint64_t cap) {
    return guarded([&] {
        std::vector<uint64_t> d;
        std::vector<double> p;
        host::load_model(path, d, *act, p);
        if (static_cast<uint64_t>(*nd) < d.size()) throw std::runtime_error("load_model: dims buffer too small");
        if (p.size() > cap) throw std::runtime_error("load_model: params buffer too small");
        *nd = static_cast<int>(d.size());
        std::memcpy(dims, d.data(), d.size() * 8);
        std::memcpy(params, p.data(), p.size() * 8);
    });
}

int parnn_allreduce_average_host(const double* c, uint64_t m, uint64_t len, double* out) {
    return guarded([&] {
        if (m == 0) throw std::runtime_error("allreduce_average: m must be >= 1");
        std::vector<const double*> v;
        for (uint64_t r = 0; r < m; ++r) v.push_back(c + r * len);
        const auto a = host::allreduce_average(v, len);
        std::memcpy(out, a.data(), len * 8);
    });
}

int parnn_ctx_create(int device, parnn_ctx** out) {
    return guarded([&] {
        auto* c = new parnn_ctx;
        c->c.reset(new Context(device));
        *out = c;
    });
}

int parnn_ctx_destroy(parnn_ctx* c) {
    return guarded([&] { delete c; });
}

int parnn_ctx_sync(parnn_ctx* c) {
    return guarded([&] { CUDA_THROW(cudaDeviceSynchronize()); });
}

int parnn_dataset_create(parnn_ctx* ctx, const double* x, const int32_t* y, uint64_t n, uint64_t d, uint64_t classes,
                         parnn_dataset** out) {
    return guarded([&] {
        need(ctx, "dataset");
        auto* p = new parnn_dataset;
        p->d.reset(new DeviceDataset(ctx->c.get(), x, y, static_cast<long>(n), static_cast<long>(d),
                                     static_cast<long>(classes)));
        *out = p;
    });
}

int parnn_dataset_destroy(parnn_dataset* ds) {
    return guarded([&] { delete ds; });
}

int parnn_dataset_generate(parnn_ctx* ctx, uint64_t classes, uint64_t dim, uint64_t per_class, double sep,
                           uint64_t seed, double cv_fraction, uint64_t split_seed, int standardize,
                           parnn_dataset** train, parnn_dataset** cv) {
    return guarded([&] {
        need(ctx, "dataset");
        need(train, "train dataset");
        need(cv, "cv dataset");
        DeviceDataset *tr = nullptr, *cvd = nullptr;
        generate_device(ctx->c.get(), classes, dim, per_class, sep, seed, cv_fraction, split_seed, standardize != 0,
                        &tr, &cvd);
        auto* a = new parnn_dataset;
        a->d.reset(tr);
        auto* b = new parnn_dataset;
        b->d.reset(cvd);
        *train = a;
        *cv = b;
    });
}

int parnn_dataset_info(parnn_dataset* ds, uint64_t* n, uint64_t* d, uint64_t* classes) {
    return guarded([&] {
        need(ds, "dataset");
        if (n) *n = static_cast<uint64_t>(ds->d->n);
        if (d) *d = static_cast<uint64_t>(ds->d->d);
        if (classes) *classes = static_cast<uint64_t>(ds->d->classes);
    });
}

int parnn_dataset_download(parnn_dataset* ds, float* x, int32_t* y) {
    return guarded([&] {
        need(ds, "dataset");
        DeviceDataset& D = *ds->d;
        CUDA_THROW(cudaSetDevice(D.ctx->device));
        CUDA_THROW(cudaDeviceSynchronize());
        if (x && D.n)
            CUDA_THROW(cudaMemcpy2D(x, D.d * 4, D.x32, D.ld * 4, D.d * 4, D.n, cudaMemcpyDeviceToHost));
        if (y && D.n) CUDA_THROW(cudaMemcpy(y, D.y, D.n * 4, cudaMemcpyDeviceToHost));
    });
}

int parnn_load_csv(const char* path, double* x, int32_t* y, uint64_t cap_rows, uint64_t cap_dim, uint64_t* n,
                   uint64_t* d, uint64_t* classes) {
    return guarded([&] {
        need(path, "load_csv path");
        uint64_t k = 0;
        const host::HostData h = host::load_csv(path, &k);
        if (n) *n = h.n;
        if (d) *d = h.d;
        if (classes) *classes = k;
        if (x && y && h.n <= cap_rows && h.d <= cap_dim) {
            std::memcpy(x, h.x.data(), h.x.size() * 8);
            std::memcpy(y, h.y.data(), h.y.size() * 4);
        }
    });
}

int parnn_dataset_load_csv(parnn_ctx* ctx, const char* path, parnn_dataset** out) {
    return guarded([&] {
        need(ctx, "dataset");
        need(path, "load_csv path");
        uint64_t k = 0;
        const host::HostData h = host::load_csv(path, &k);
        auto* p = new parnn_dataset;
        p->d.reset(new DeviceDataset(ctx->c.get(), h.x.data(), h.y.data(), static_cast<long>(h.n),
                                     static_cast<long>(h.d), static_cast<long>(k)));
        *out = p;
    });
}

int parnn_save_csv(const char* path, const double* x, const int32_t* y, uint64_t n, uint64_t d) {
    return guarded([&] {
        need(path, "save_csv path");
        host::HostData h;
        h.n = n;
        h.d = d;
        h.x.assign(x, x + n * d);
        h.y.assign(y, y + n);
        host::save_csv(path, h);
    });
}

int parnn_replica_create(parnn_ctx* ctx, const uint64_t* dims, int nd, int act, int prec, int opt, uint64_t minibatch,
                         uint64_t max_steps, double decay, double smoothing, parnn_replica** out) {
    return guarded([&] {
        need(ctx, "replica");
        if (decay <= 0.0 || decay >= 1.0)
            throw std::runtime_error("ng_init: decay must be in (0,1), got " + host::fmt_num(decay));
        if (smoothing <= 0.0) throw std::runtime_error("ng_init: smoothing must be positive, got " + host::fmt_num(smoothing));
        if (opt < 0 || opt > 2) throw std::runtime_error("replica: unknown optimizer " + std::to_string(opt));
        auto* p = new parnn_replica;
        p->r.reset(new Replica(ctx->c.get(), to_dims(dims, nd), act, static_cast<Precision>(prec),
                               static_cast<Optimizer>(opt), static_cast<long>(minibatch), static_cast<long>(max_steps),
                               decay, smoothing));
        *out = p;
    });
}

int parnn_replica_set_lowrank(parnn_replica* r, int rank_in, int rank_out, int update_period, int init_iters,
                              double history, int update_lag) {
    return guarded([&] {
        need(r, "replica");
        LrConfig c = r->r->lrc;
        c.rank_in = rank_in;
        c.rank_out = rank_out;
        c.update_period = update_period;
        c.init_iters = init_iters;
        c.history = history;
        c.update_lag = update_lag;
        r->r->set_lowrank(c);
    });
}

int parnn_replica_lowrank_state(parnn_replica* r, int layer, int side, double* w, double* d, double* rho,
                                uint64_t* rank, uint64_t* dim) {
    return guarded([&] {
        need(r, "replica");
        Replica& rp = *r->r;
        if (rp.opt != OPT_NG_LOWRANK) throw std::runtime_error("replica: not a low-rank NG-SGD replica");
        if (layer < 0 || layer >= rp.L || side < 0 || side > 1) throw std::runtime_error("ng lowrank: bad layer/side");
        const LrSide& sd = side == 0 ? rp.lrl[layer].in : rp.lrl[layer].out;
        if (rank) *rank = static_cast<uint64_t>(sd.R);
        if (dim) *dim = static_cast<uint64_t>(sd.D);
        rp.get_lowrank_state(layer, side, w, d, rho);
    });
}

int parnn_replica_lowrank_diag(parnn_replica* r, int layer, int side, double out[4]) {
    return guarded([&] {
        need(r, "replica");
        Replica& rp = *r->r;
        if (rp.opt != OPT_NG_LOWRANK) throw std::runtime_error("replica: not a low-rank NG-SGD replica");
        if (layer < 0 || layer >= rp.L || side < 0 || side > 1) throw std::runtime_error("ng lowrank: bad layer/side");
        const LrSide& sd = side == 0 ? rp.lrl[layer].in : rp.lrl[layer].out;
        CUDA_THROW(cudaDeviceSynchronize());
        CUDA_THROW(cudaMemcpy(out, sd.st + 2 * sd.R + 1, 6 * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int parnn_debug_lowrank_eig(int rank, uint64_t dim, double eta, double a, double alpha, const double* state_in,
                            const float* gram, double* state_out, float* m_out, int* sweeps) {
    return guarded([&] {
        if (rank < 1 || rank > LR_MAX_RANK) throw std::runtime_error("ng lowrank: bad rank");
        lr_debug_eig(rank, static_cast<long>(dim), eta, a, alpha, state_in, gram, state_out, m_out, sweeps);
    });
}

int parnn_debug_gemm(int precision, int a_mn, int b_mn, int m, int n, int k, int mode, int act, int ksplit,
                     int force_bn, int force_mc, int lower, int bias_col, float alpha, float beta, float lr,
                     const float* a, const float* b, const float* bias, const float* aux, float* out, float* out2,
                     double* sums, int* info) {
    return guarded([&] {
        need(a, "gemm A");
        need(b, "gemm B");
        need(out, "gemm out");
        if (precision < 0 || precision > 2) throw std::runtime_error("gemm: unknown precision");
        if (mode < EPI_FWD_ACT || mode > EPI_RESID) throw std::runtime_error("gemm: unknown epilogue mode");
        if ((mode == EPI_FWD_ACT || mode == EPI_FWD_LINEAR || (mode == EPI_GRAD_SGD && bias_col >= 0)) && !bias)
            throw std::runtime_error("gemm: mode needs a bias vector");
        if ((mode == EPI_ACTGRAD || mode == EPI_RESID) && !aux) throw std::runtime_error("gemm: mode needs aux");
        debug_gemm(precision, a_mn != 0, b_mn != 0, m, n, k, mode, act, ksplit, force_bn, force_mc, lower, bias_col,
                   alpha, beta, lr, a, b, bias, aux, out, out2, sums, info);
    });
}

int parnn_lowrank_basis(uint64_t dim, uint64_t rank, uint64_t seed, double* out) {
    return guarded([&] {
        const std::vector<double> b = host::lowrank_basis(dim, rank, seed);
        std::copy(b.begin(), b.end(), out);
    });
}

uint64_t parnn_lowrank_seed(int layer, int side) { return host::lowrank_seed(layer, side); }

int parnn_replica_destroy(parnn_replica* r) {
    return guarded([&] { delete r; });
}

int parnn_replica_set_params(parnn_replica* r, const double* p, uint64_t n) {
    return guarded([&] {
        if (n != flat_count(*r->r))
            throw std::runtime_error("unflatten: vector length " + std::to_string(n) + " does not match model size " +
                                     std::to_string(flat_count(*r->r)));
        r->r->set_params(p);
    });
}

int parnn_replica_get_params(parnn_replica* r, double* p, uint64_t n) {
    return guarded([&] {
        if (n < flat_count(*r->r)) throw std::runtime_error("flatten: output buffer too small");
        r->r->get_params(p);
    });
}

int parnn_replica_get_ng_state(parnn_replica* r, double* f, uint64_t n) {
    return guarded([&] {
        if (n < padded_factor_count(*r->r)) throw std::runtime_error("ng_state: output buffer too small");
        r->r->get_ng_state(f);
    });
}

int parnn_replica_set_ng_state(parnn_replica* r, const double* f, uint64_t n, uint64_t t) {
    return guarded([&] {
        if (n != padded_factor_count(*r->r)) throw std::runtime_error("ng_state: factor count mismatch");
        r->r->set_ng_state(f, static_cast<long>(t));
    });
}

int parnn_replica_bind(parnn_replica* r, parnn_dataset* ds) {
    return guarded([&] { r->r->bind(ds->d.get()); });
}

int parnn_replica_upload_epoch(parnn_replica* r, const uint32_t* rows, const float* lrs, uint64_t steps) {
    return guarded([&] {
        Replica& R = *r->r;
        if (!R.bound) throw std::runtime_error("replica: bind a dataset first");
        for (uint64_t i = 0; i < steps * R.B; ++i)
            if (rows[i] >= static_cast<uint64_t>(R.bound->n))
                throw std::runtime_error("Dataset::select: index " + std::to_string(rows[i]) + " out of range " +
                                         std::to_string(R.bound->n));
        for (uint64_t i = 0; i < steps; ++i)
            if (lrs[i] < 0.f) throw std::runtime_error("sgd_step: negative learning rate " + host::fmt_num(lrs[i]));
        R.upload_epoch(rows, lrs, static_cast<long>(steps));
    });
}

int parnn_replica_step(parnn_replica* r, uint64_t steps) {
    return guarded([&] {
        for (uint64_t i = 0; i < steps; ++i) r->r->run_step(r->r->stream);
    });
}

int parnn_replica_sync(parnn_replica* r) {
    return guarded([&] { r->r->check_errors(); });
}

int parnn_replica_ce(parnn_replica* r, double* out, uint64_t steps) {
    return guarded([&] {
        CUDA_THROW(cudaStreamSynchronize(r->r->stream));
        CUDA_THROW(cudaMemcpy(out, r->r->d_ce, steps * 8, cudaMemcpyDeviceToHost));
    });
}

int parnn_replica_step_ce(parnn_replica* r, uint64_t step, double* out) {
    return guarded([&] { *out = r->r->step_ce(static_cast<long>(step)); });
}

int parnn_replica_forward(parnn_replica* r, parnn_dataset* ds, const uint32_t* rows, uint64_t b, float* z) {
    return guarded([&] {
        if (!r->r->bound) r->r->bind(ds->d.get());
        r->r->forward_only(ds->d.get(), rows, static_cast<long>(b), z);
    });
}

int parnn_replica_accuracy(parnn_replica* r, parnn_dataset* ds, double* acc) {
    return guarded([&] { *acc = r->r->accuracy(ds->d.get()); });
}

int parnn_replica_kernels_per_step(parnn_replica* r, uint64_t* n) {
    return guarded([&] {
        Replica& R = *r->r;
        if (!R.graph && R.kernels_per_step == 0) throw std::runtime_error("replica: no step graph");
        *n = static_cast<uint64_t>(R.kernels_per_step);
    });
}

int parnn_replica_time_steps(parnn_replica* r, uint64_t steps, double* ms) {
    return guarded([&] { *ms = r->r->time_steps(static_cast<long>(steps)); });
}

int parnn_replica_profile(parnn_replica* r, uint64_t steps, char* names, uint64_t names_cap, double* ms,
                          double* flops, uint64_t cap, uint64_t* n_regions) {
    return guarded([&] {
        std::vector<std::string> nm;
        std::vector<double> t, f;
        r->r->profile_steps(static_cast<long>(steps), nm, t, f);
        std::string joined;
        for (auto& x : nm) joined += x + "\n";
        if (joined.size() + 1 > names_cap || nm.size() > cap) throw std::runtime_error("profile: buffers too small");
        std::memcpy(names, joined.c_str(), joined.size() + 1);
        for (size_t i = 0; i < nm.size(); ++i) {
            ms[i] = t[i];
            flops[i] = f[i];
        }
        *n_regions = nm.size();
    });
}

int parnn_run_steps(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total, uint64_t steps,
                    uint64_t avg_frequency, double* ms) {
    return guarded([&] {
        if (n_local <= 0) throw std::runtime_error("run_steps: no replicas");
        if (avg_frequency == 0) throw std::runtime_error("train_parallel: avg_frequency must be >= 1");
        std::vector<Replica*> v;
        for (int i = 0; i < n_local; ++i) v.push_back(reps[i]->r.get());
        Context* ctx = v[0]->ctx;
        Averager avg(ctx, v, comm ? comm->c.get() : nullptr, static_cast<long>(m_total));
        cudaEvent_t a, b;
        CUDA_THROW(cudaEventCreate(&a));
        CUDA_THROW(cudaEventCreate(&b));
        for (Replica* r : v) CUDA_THROW(cudaStreamSynchronize(r->stream));
        CUDA_THROW(cudaEventRecord(a, ctx->stream));
        for (Replica* r : v) CUDA_THROW(cudaStreamWaitEvent(r->stream, a, 0));
        for (uint64_t s = 0; s < steps; ++s) {
            const bool window_end = (s + 1) % avg_frequency == 0 || s + 1 == steps;  // last event closes the window
            for (Replica* r : v) r->run_step(r->stream, window_end);
            if (window_end) avg.run();
        }
        // join: every replica stream (the last step's tail) and the averaging stream
        std::vector<cudaEvent_t> tails(v.size() + 1);
        for (size_t i = 0; i < tails.size(); ++i) {
            CUDA_THROW(cudaEventCreateWithFlags(&tails[i], cudaEventDisableTiming));
            CUDA_THROW(cudaEventRecord(tails[i], i < v.size() ? v[i]->stream : ctx->avg));
            CUDA_THROW(cudaStreamWaitEvent(ctx->stream, tails[i], 0));
        }
        CUDA_THROW(cudaEventRecord(b, ctx->stream));
        for (auto e : tails) cudaEventDestroy(e);
        CUDA_THROW(cudaEventSynchronize(b));
        float t = 0.f;
        CUDA_THROW(cudaEventElapsedTime(&t, a, b));
        *ms = t;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int parnn_averager_create(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total,
                          parnn_averager** out) {
    return guarded([&] {
        if (n_local <= 0) throw std::runtime_error("allreduce_average: m must be >= 1");
        std::vector<Replica*> v;
        for (int i = 0; i < n_local; ++i) v.push_back(reps[i]->r.get());
        auto* p = new parnn_averager;
        p->a.reset(new Averager(v[0]->ctx, v, comm ? comm->c.get() : nullptr, static_cast<long>(m_total)));
        *out = p;
    });
}

int parnn_averager_run(parnn_averager* a) {
    return guarded([&] {
        need(a, "averager");
        a->a->run();
    });
}

int parnn_averager_destroy(parnn_averager* a) {
    return guarded([&] {
        if (a) CUDA_THROW(cudaStreamSynchronize(a->a->ctx->avg));
        delete a;
    });
}

int parnn_time_average(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total, uint64_t iters,
                       double* ms, double* bytes) {
    return guarded([&] {
        if (n_local <= 0) throw std::runtime_error("allreduce_average: m must be >= 1");
        std::vector<Replica*> v;
        for (int i = 0; i < n_local; ++i) v.push_back(reps[i]->r.get());
        Context* ctx = v[0]->ctx;
        Averager avg(ctx, v, comm ? comm->c.get() : nullptr, static_cast<long>(m_total));
        for (Replica* r : v) CUDA_THROW(cudaStreamSynchronize(r->stream));
        avg.run();  // warm (NCCL channels, first-touch)
        cudaEvent_t a, b;
        CUDA_THROW(cudaEventCreate(&a));
        CUDA_THROW(cudaEventCreate(&b));
        CUDA_THROW(cudaEventRecord(a, ctx->avg));
        for (uint64_t i = 0; i < iters; ++i) avg.run();
        CUDA_THROW(cudaEventRecord(b, ctx->avg));
        CUDA_THROW(cudaEventSynchronize(b));
        float t = 0.f;
        CUDA_THROW(cudaEventElapsedTime(&t, a, b));
        *ms = t / static_cast<double>(std::max<uint64_t>(iters, 1));
        *bytes = avg.bytes();
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int parnn_dataset_write_f32(parnn_dataset* ds, const float* x, const int32_t* y, uint64_t row0, uint64_t n) {
    return guarded([&] { ds->d->write_rows(x, y, static_cast<long>(row0), static_cast<long>(n), ds->d->ctx->stream); });
}

int parnn_comm_unique_id(unsigned char out[128]) {
    return guarded([&] { nccl_unique_id(out); });
}

int parnn_comm_create(parnn_ctx* ctx, const unsigned char id[128], int nranks, int rank, parnn_comm** out) {
    return guarded([&] {
        auto* p = new parnn_comm;
        p->c.reset(new Comm(ctx->c.get(), id, nranks, rank));
        *out = p;
    });
}

int parnn_comm_destroy(parnn_comm* c) {
    return guarded([&] { delete c; });
}

int parnn_average(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total) {
    return guarded([&] {
        if (n_local <= 0) throw std::runtime_error("allreduce_average: m must be >= 1");
        std::vector<Replica*> v;
        for (int i = 0; i < n_local; ++i) v.push_back(reps[i]->r.get());
        Averager a(v[0]->ctx, v, comm ? comm->c.get() : nullptr, static_cast<long>(m_total));
        a.run();
        for (Replica* r : v) CUDA_THROW(cudaStreamSynchronize(r->stream));
        CUDA_THROW(cudaStreamSynchronize(v[0]->ctx->avg));
    });
}

int parnn_train(parnn_ctx* ctx, parnn_comm* comm, const parnn_train_config* c, const uint64_t* dims, int nd,
                const double* params0, parnn_dataset* train_set, parnn_dataset* cv, double* params_out,
                double* metrics_out, uint64_t* epochs_run) {
    return guarded([&] {
        need(ctx, "train");
        need(train_set, "train dataset");
        need(c, "train config");
        TrainConfig t;
        t.workers = c->workers;
        t.avg_frequency = c->avg_frequency;
        t.minibatch = c->minibatch;
        t.base_seed = c->base_seed;
        t.optimizer = c->optimizer;
        t.newbob = c->lr_schedule == PARNN_NEWBOB;
        t.lr_init = c->lr_init;
        t.epochs = c->epochs;
        t.ng_decay = c->ng_decay;
        t.ng_smoothing = c->ng_smoothing;
        t.precision = c->precision;
        t.activation = c->activation;
        t.rank0 = c->rank0;
        t.local = c->local_workers;
        t.serial = c->serial;
        if (c->optimizer < 0 || c->optimizer > 2)
            throw std::runtime_error("train_parallel: unknown optimizer " + std::to_string(c->optimizer));
        if (c->ng_rank_in) t.lr.rank_in = c->ng_rank_in;
        if (c->ng_rank_out) t.lr.rank_out = c->ng_rank_out;
        if (c->ng_update_period) t.lr.update_period = c->ng_update_period;
        if (c->ng_history > 0.0) t.lr.history = c->ng_history;
        if (c->ng_update_lag) t.lr.update_lag = c->ng_update_lag;
        std::vector<EpochRec> met;
        pnb::train(ctx->c.get(), comm ? comm->c.get() : nullptr, t, to_dims(dims, nd), params0, train_set->d.get(),
              cv ? cv->d.get() : nullptr, params_out, met);
        for (size_t e = 0; e < met.size(); ++e) {
            const EpochRec& m = met[e];
            double* row = metrics_out + 7 * e;
            row[0] = m.epoch;
            row[1] = m.lr;
            row[2] = m.train_ce;
            row[3] = m.cv_accuracy;
            row[4] = m.wall_seconds;
            row[5] = m.workers;
            row[6] = m.avg_events;
        }
        *epochs_run = met.size();
    });
}

int parnn_rbm_create(parnn_ctx* ctx, uint64_t v, uint64_t h, int gaussian, uint64_t batch, int prec, parnn_rbm** out) {
    return guarded([&] {
        auto* p = new parnn_rbm;
        p->r.reset(new RbmDevice(ctx->c.get(), static_cast<long>(v), static_cast<long>(h), gaussian != 0,
                                 static_cast<long>(batch), static_cast<Precision>(prec)));
        *out = p;
    });
}

int parnn_rbm_destroy(parnn_rbm* r) {
    return guarded([&] { delete r; });
}

int parnn_rbm_set_params(parnn_rbm* r, const double* p) {
    return guarded([&] { r->r->set_params(p); });
}

int parnn_rbm_get_params(parnn_rbm* r, double* p) {
    return guarded([&] { r->r->get_params(p); });
}

int parnn_rbm_cd1(parnn_rbm* r, const double* batch, uint64_t b, double lr, int sampling, uint64_t seed,
                  uint64_t counter, const double* u) {
    return guarded([&] { r->r->cd1_host(batch, static_cast<long>(b), lr, sampling, seed, counter, u); });
}

int parnn_rbm_hidden_probs(parnn_rbm* r, const double* x, uint64_t n, double* out) {
    return guarded([&] { r->r->hidden_probs_host(x, static_cast<long>(n), out); });
}

int parnn_rbm_reconstruction_error(parnn_rbm* r, const double* x, uint64_t n, double* out) {
    return guarded([&] { *out = r->r->reconstruction_error_host(x, static_cast<long>(n)); });
}

int parnn_greedy_pretrain(parnn_ctx* ctx, const uint64_t* dims, int nd, const double* data, uint64_t n, uint64_t epochs,
                          double lr_g, double lr_b, uint64_t batch, uint64_t seed, int prec, double* params_out) {
    return guarded([&] {
        host::Rng rng(seed);
        greedy_pretrain(ctx->c.get(), to_dims(dims, nd), data, static_cast<long>(n), epochs, lr_g, lr_b,
                        static_cast<long>(batch), rng, seed ^ 0x5851F42D4C957F2Dull, static_cast<Precision>(prec),
                        params_out);
    });
}

int parnn_greedy_pretrain_rng(parnn_ctx* ctx, const uint64_t* dims, int nd, const double* data, uint64_t n,
                              uint64_t epochs, double lr_g, double lr_b, uint64_t batch, int activation,
                              uint64_t rng_state[4], double* rng_spare, int* rng_has_spare, int prec,
                              double* params_out) {
    return guarded([&] {
        need(ctx, "greedy_pretrain");
        need(rng_state, "greedy_pretrain rng state");
        need(rng_spare, "greedy_pretrain rng spare");
        need(rng_has_spare, "greedy_pretrain rng spare flag");
        if (activation != PARNN_SIGMOID && activation != PARNN_TANH)
            throw std::runtime_error("greedy_pretrain: unknown activation " + std::to_string(activation));
        host::Rng rng(0);
        rng.set_state(rng_state, *rng_spare, *rng_has_spare != 0);
        // the device Bernoulli stream is keyed by the caller's generator state on entry
        uint64_t key = 0x5851F42D4C957F2Dull;
        for (int i = 0; i < 4; ++i) key = (key ^ rng_state[i]) * 0x9E3779B97F4A7C15ull;
        greedy_pretrain(ctx->c.get(), to_dims(dims, nd), data, static_cast<long>(n), epochs, lr_g, lr_b,
                        static_cast<long>(batch), rng, key, static_cast<Precision>(prec), params_out);
        bool has = false;
        rng.get_state(rng_state, rng_spare, &has);
        *rng_has_spare = has ? 1 : 0;
    });
}

int parnn_pretrain_last_stats(double* cd1_device_seconds, uint64_t* cd1_steps, double* cd1_flop) {
    return guarded([&] {
        if (cd1_device_seconds) *cd1_device_seconds = g_pretrain_stats.cd1_seconds;
        if (cd1_steps) *cd1_steps = g_pretrain_stats.cd1_steps;
        if (cd1_flop) *cd1_flop = g_pretrain_stats.cd1_flop;
    });
}

}  // extern "C"
