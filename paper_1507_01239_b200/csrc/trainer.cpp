// The model-averaging train loop (parallel.cpp:97-275) for the workers one
// process hosts on its GPU. Host logic (sharding, per-worker RNG streams,
// minibatch order, LR schedule, averaging triggers, metrics) follows the
// reference exactly; all arithmetic runs on the device.
#include <algorithm>
#include <chrono>
#include <memory>

#include "host.h"
#include "parallel.h"

namespace pnb {

void train(Context* ctx, Comm* comm, const TrainConfig& cfg, const std::vector<long>& dims, const double* params0,
           DeviceDataset* train_ds, DeviceDataset* cv_ds, double* params_out, std::vector<EpochRec>& metrics,
           double* step_seconds) {
    if (cfg.workers == 0) throw std::runtime_error("train_parallel: workers must be >= 1");
    if (cfg.avg_frequency == 0) throw std::runtime_error("train_parallel: avg_frequency must be >= 1");
    if (cfg.minibatch == 0) throw std::runtime_error("train_parallel: minibatch must be >= 1");
    if (cfg.epochs > 0 && (!cv_ds || cv_ds->n == 0)) throw std::runtime_error("train_parallel: empty CV set");
    const uint64_t m = cfg.workers;
    // placement: without a communicator this process hosts every worker; with one,
    // each of the comm's processes hosts the contiguous block [rank * m/n, (rank+1) * m/n)
    uint64_t local = cfg.local;
    if (!comm) {
        if (local == 0) local = m;
        if (local != m || cfg.rank0 != 0)
            throw std::runtime_error("train_parallel: without a communicator this process must host all " +
                                     std::to_string(m) + " workers (got " + std::to_string(local) + " from rank " +
                                     std::to_string(cfg.rank0) + ")");
    } else {
        const uint64_t nr = static_cast<uint64_t>(comm->nranks);
        if (m % nr != 0)
            throw std::runtime_error("train_parallel: " + std::to_string(m) + " workers do not split over " +
                                     std::to_string(nr) + " processes");
        if (local == 0) local = m / nr;
        if (local != m / nr || cfg.rank0 != static_cast<uint64_t>(comm->rank) * local)
            throw std::runtime_error("train_parallel: process " + std::to_string(comm->rank) + " must host workers [" +
                                     std::to_string(comm->rank * (m / nr)) + ", " +
                                     std::to_string((comm->rank + 1) * (m / nr)) + ")");
    }

    // partition_data: one global shuffle by base_seed, m contiguous shards.
    const std::vector<uint64_t> shards = host::partition_rows(train_ds->n, m, cfg.base_seed);
    const uint64_t S = train_ds->n / m;
    const uint64_t B = cfg.minibatch;
    const uint64_t nb = B <= S ? S / B : 0;
    // ng_init runs for every worker whatever the optimizer (parallel.cpp:178)
    if (cfg.ng_decay <= 0.0 || cfg.ng_decay >= 1.0)
        throw std::runtime_error("ng_init: decay must be in (0,1), got " + host::fmt_num(cfg.ng_decay));
    if (cfg.ng_smoothing <= 0.0)
        throw std::runtime_error("ng_init: smoothing must be positive, got " + host::fmt_num(cfg.ng_smoothing));
    host::Schedule sched = host::make_schedule(cfg.newbob != 0, cfg.lr_init, cfg.epochs);
    const host::Schedule exp_sched = host::make_schedule(false, cfg.lr_init, cfg.epochs);
    if (cfg.epochs > 0 && B > S) {  // raised by minibatches() inside worker_epoch (data.cpp:188-191)
        const std::string msg =
            "minibatches: batch size " + std::to_string(B) + " exceeds dataset size " + std::to_string(S);
        if (cfg.serial) throw std::runtime_error(msg);
        throw std::runtime_error("train_parallel: worker rank " + std::to_string(cfg.rank0) + " failed: " + msg);
    }

    std::vector<std::unique_ptr<Replica>> owned;
    std::vector<Replica*> reps;
    std::vector<host::Rng> rngs;
    for (uint64_t i = 0; i < local; ++i) {
        owned.emplace_back(new Replica(ctx, dims, cfg.activation, static_cast<Precision>(cfg.precision),
                                       static_cast<Optimizer>(cfg.optimizer), static_cast<long>(B),
                                       static_cast<long>(std::max<uint64_t>(nb, 1)), cfg.ng_decay, cfg.ng_smoothing));
        if (cfg.optimizer == OPT_NG_LOWRANK) {
            LrConfig lc = cfg.lr;
            lc.alpha = cfg.ng_smoothing;
            owned.back()->set_lowrank(lc);
        }
        reps.push_back(owned.back().get());
        reps.back()->set_params(params0);
        reps.back()->bind(train_ds);
        rngs.emplace_back(cfg.base_seed + cfg.rank0 + i);  // Rng(base_seed + rank)
    }
    Averager avg(ctx, reps, comm, static_cast<long>(m));

    double prev_acc = 0.0;
    bool have_prev = false;
    std::vector<uint32_t> rows(nb * B);
    std::vector<float> lrs(std::max<uint64_t>(nb, 1));
    std::vector<double> ce(std::max<uint64_t>(nb, 1));

    for (uint64_t epoch = 0; epoch < cfg.epochs; ++epoch) {
        const double newbob_lr = sched.newbob_lr;
        for (uint64_t b = 0; b < nb; ++b) {
            double lr = newbob_lr;
            if (!cfg.newbob) {
                double progress = (static_cast<double>(epoch) + static_cast<double>(b) / static_cast<double>(nb)) /
                                  static_cast<double>(cfg.epochs);
                if (progress > 1.0) progress = 1.0;
                lr = host::exponential_lr(exp_sched, progress);
            }
            lrs[b] = static_cast<float>(lr);
        }
        for (uint64_t i = 0; i < local; ++i) {
            const uint64_t rank = cfg.rank0 + i;
            const uint64_t seed = rngs[i].next_u64();  // worker_epoch: minibatches(shard, B, rng.next_u64())
            const std::vector<uint64_t> pos = host::minibatch_rows(S, B, seed);
            for (uint64_t j = 0; j < nb * B; ++j) rows[j] = static_cast<uint32_t>(shards[rank * S + pos[j]]);
            reps[i]->upload_epoch(rows.data(), lrs.data(), static_cast<long>(nb));
        }
        for (Replica* r : reps) CUDA_THROW(cudaStreamSynchronize(r->stream));
        const auto t0 = std::chrono::steady_clock::now();

        uint64_t since = 0, events = 0;
        for (uint64_t b = 0; b < nb; ++b) {
            // the step that closes an averaging window (K-th, or the epoch's last: forced
            // average) records its per-layer update events for the bucketed average
            const bool window_end = since + 1 == cfg.avg_frequency || b + 1 == nb;
            for (Replica* r : reps) r->run_step(r->stream, window_end);
            if (++since == cfg.avg_frequency) {
                avg.run();
                since = 0;
                ++events;
            }
        }
        if (since > 0) {  // forced epoch-boundary averaging (parallel.cpp:140-144)
            avg.run();
            ++events;
        }
        for (Replica* r : reps) CUDA_THROW(cudaStreamSynchronize(r->stream));
        CUDA_THROW(cudaStreamSynchronize(ctx->avg));
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (step_seconds && nb) *step_seconds = wall / static_cast<double>(nb);

        for (size_t i = 0; i < reps.size(); ++i) {
            try {
                reps[i]->check_errors();
            } catch (const std::exception& e) {
                if (cfg.serial) throw;
                throw std::runtime_error("train_parallel: worker rank " + std::to_string(cfg.rank0 + i) +
                                         " failed: " + e.what());
            }
        }
        double ce_sum = 0.0;
        for (Replica* r : reps) {
            if (nb) CUDA_THROW(cudaMemcpy(ce.data(), r->d_ce, nb * sizeof(double), cudaMemcpyDeviceToHost));
            for (uint64_t b = 0; b < nb; ++b) ce_sum += ce[b];
        }
        if (comm) ce_sum = comm->allreduce_sum(ce_sum);
        const double cv_acc = reps[0]->accuracy(cv_ds);

        EpochRec rec;
        rec.epoch = static_cast<double>(epoch + 1);
        rec.lr = cfg.newbob ? newbob_lr
                            : host::exponential_lr(sched, static_cast<double>(epoch) / static_cast<double>(cfg.epochs));
        rec.train_ce = nb ? ce_sum / static_cast<double>(nb * m) : 0.0;
        rec.cv_accuracy = cv_acc;
        rec.wall_seconds = wall;
        rec.workers = static_cast<double>(m);
        rec.avg_events = static_cast<double>(events);
        metrics.push_back(rec);

        if (cfg.newbob && have_prev) {
            if (host::newbob_next(sched, prev_acc, cv_acc, nullptr)) {
                prev_acc = cv_acc;
                break;
            }
        }
        prev_acc = cv_acc;
        have_prev = true;
    }
    reps[0]->get_params(params_out);
}

}  // namespace pnb
