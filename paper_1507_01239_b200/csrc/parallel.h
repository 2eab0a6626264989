// Cross-replica averaging and the multi-GPU communicator (NCCL over NVLink).
#pragma once
#include <cstring>
#include <vector>

#include "runtime.h"

namespace pnb {

struct Comm {
    Context* ctx;
    void* comm = nullptr;  // ncclComm_t
    int nranks = 1, rank = 0;
    double* dscratch = nullptr;
    Comm(Context* c, const unsigned char id[128], int nranks, int rank);
    ~Comm();
    double allreduce_sum(double v);
};

void nccl_unique_id(unsigned char out[128]);

// Replaces every local replica's parameters with the mean over all m workers
// (local replicas + every other process in `comm`), one layer bucket
// ([W_l | b_l]) at a time on the context stream, in the order the averaged step
// finishes the layers (L-1 .. 0): bucket l starts when every local replica has
// recorded ev_upd[l] and ends by recording each replica's ev_gate[l], which the
// replica's next forward of layer l waits on (runtime.h).
struct Averager {
    Context* ctx;
    std::vector<Replica*> reps;
    Comm* comm;
    long m_total;
    long n = 0;
    float** d_src = nullptr;
    bf16** d_shadow = nullptr;
    bf16** d_null_shadow = nullptr;  // one null shadow pointer: the unscaled partial sum has none
    float* scratch = nullptr;
    float** d_scratch_ptr = nullptr;
    bool work = false;  // false: one local replica, no communicator, m = 1 -- the identity
    Averager(Context* c, const std::vector<Replica*>& reps, Comm* comm, long m_total);
    ~Averager();
    void run();
    // bytes one averaging event moves per GPU over the interconnect (fp32 params)
    double bytes() const { return 4.0 * static_cast<double>(n); }
};

struct TrainConfig {
    uint64_t workers = 1, avg_frequency = 10, minibatch = 128, base_seed = 0;
    int optimizer = 1;   // 0 sgd, 1 ngsgd kron-full (parallel.hpp:31-38 default), 2 ngsgd low-rank
    int newbob = 0;      // 0 exponential (default), 1 newbob
    double lr_init = 0.32;
    uint64_t epochs = 15;
    double ng_decay = 0.95, ng_smoothing = 4.0;
    int precision = PREC_BF16;
    int activation = 0;
    uint64_t rank0 = 0;   // first global worker rank hosted by this process
    uint64_t local = 0;   // workers hosted by this process (0 = all)
    int serial = 0;       // serial_train semantics (errors not wrapped)
    LrConfig lr;          // optimizer 2: low-rank NG-SGD knobs (alpha = ng_smoothing)
};

struct EpochRec {
    double epoch, lr, train_ce, cv_accuracy, wall_seconds, workers, avg_events;
};

// train_loop (parallel.cpp:163-275) for the workers this process hosts.
void train(Context* ctx, Comm* comm, const TrainConfig& cfg, const std::vector<long>& dims, const double* params0,
           DeviceDataset* train_ds, DeviceDataset* cv_ds, double* params_out, std::vector<EpochRec>& metrics,
           double* step_seconds = nullptr);

}  // namespace pnb
