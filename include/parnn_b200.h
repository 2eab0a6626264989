/*
 * parnn_b200 — C ABI of the B200-native model-averaging DNN trainer.
 *
 * Drop-in boundary for the reference's trainer path (namespace parnn in
 * /root/reference/proj). The reference has no FFI of its own; every entry
 * point below names the reference interface it replaces (file:line). All
 * functions return PARNN_OK (0) or PARNN_ERR (-1); on error
 * parnn_last_error() returns the message (thread-local), whose text follows
 * the reference's parnn::Error message for the same condition.
 *
 * Conventions: model parameters are fp64 host vectors in the reference's
 * canonical flatten order [W0 row-major, b0, W1, b1, ...]
 * (network.hpp:59-66); matrices are row-major fp64; labels int32.
 */
#ifndef PARNN_B200_H
#define PARNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARNN_OK 0
#define PARNN_ERR (-1)

/* GEMM operand precision (fp32 accumulation always): BF16, TF32, or FP32 =
 * fp32-accurate 3xTF32 split on the tensor cores (the parity mode). */
enum parnn_precision { PARNN_BF16 = 0, PARNN_TF32 = 1, PARNN_FP32 = 2 };
/* parallel.hpp:14-18. PARNN_NGSGD is the reference's kron-full NG-SGD
 * (optimizer.cpp:44-157); PARNN_NGSGD_LOWRANK is the north star's online
 * low-rank NG-SGD (not in the reference, oracle/ng_lowrank.py). */
enum parnn_optimizer { PARNN_SGD = 0, PARNN_NGSGD = 1, PARNN_NGSGD_LOWRANK = 2 };
enum parnn_lr_variant { PARNN_NEWBOB = 0, PARNN_EXPONENTIAL = 1 }; /* optimizer.hpp:57 */
enum parnn_activation { PARNN_SIGMOID = 0, PARNN_TANH = 1 };   /* network.hpp:16 */

typedef struct parnn_ctx parnn_ctx;
typedef struct parnn_dataset parnn_dataset;
typedef struct parnn_replica parnn_replica;
typedef struct parnn_comm parnn_comm;
typedef struct parnn_rbm parnn_rbm;

const char* parnn_last_error(void);
const char* parnn_version(void);

/* ---------------- host primitives (bit-exact with the reference) -------- */
/* Rng::next_u64 stream (rng.cpp:30-41, seeded rng.cpp:25-28) */
int parnn_rng_u64(uint64_t seed, uint64_t n, uint64_t* out);
/* Rng::uniform (rng.cpp:43-45) */
int parnn_rng_uniform(uint64_t seed, uint64_t n, double* out);
/* Rng::gaussian_vector (rng.cpp:60-84) */
int parnn_rng_gaussian(uint64_t seed, uint64_t n, double mean, double stddev, double* out);
/* shuffled_indices (data.cpp:162-168, data.hpp:53-55) */
int parnn_shuffled_indices(uint64_t n, uint64_t seed, uint64_t* out);
/* partition_data (parallel.cpp:61-77): m*floor(n/m) row ids, shard-major */
int parnn_partition_rows(uint64_t n, uint64_t m, uint64_t seed, uint64_t* out);
/* minibatches (data.cpp:185-203): floor(n/b)*b shard positions, batch-major */
int parnn_minibatch_rows(uint64_t n, uint64_t b, uint64_t seed, uint64_t* out);
/* generate_synthetic + split_cv + feature_stats/standardize_in_place
 * (data.cpp:124-242); buffers sized classes*per_class rows. */
int parnn_make_data(uint64_t classes, uint64_t dim, uint64_t per_class, double separation, uint64_t seed,
                    double cv_fraction, uint64_t split_seed, int standardize, double* train_x, int32_t* train_y,
                    uint64_t* n_train, double* cv_x, int32_t* cv_y, uint64_t* n_cv);
/* param_count (network.cpp:32-38) */
uint64_t parnn_param_count(const uint64_t* dims, int ndims);
/* init_random (network.cpp:40-60) with Rng(seed) */
int parnn_init_random(const uint64_t* dims, int ndims, uint64_t seed, double* params);
/* exponential_lr (optimizer.cpp:198-203) */
int parnn_exponential_lr(double lr_init, uint64_t planned_epochs, double progress, double* lr);
/* newbob_next (optimizer.cpp:181-196) over a CV-accuracy sequence: lr/stop per epoch >= 2 */
int parnn_newbob_sequence(double lr_init, const double* accs, uint64_t n, double* lr_out, int* stop_out);
/* scale_lr_for_workers (optimizer.cpp:205-208) */
int parnn_scale_lr_for_workers(double lr_init, uint64_t workers, double* lr);
/* save_model / load_model, PARNNET1 (network.cpp:291-369) */
int parnn_save_model(const char* path, const uint64_t* dims, int ndims, int activation, const double* params);
int parnn_load_model(const char* path, uint64_t* dims, int* ndims, int* activation, double* params,
                     uint64_t capacity);
/* Low-rank NG initial basis: rank x dim, orthonormal rows (Rng(seed) gaussians,
 * modified Gram-Schmidt). Seeds per (layer, side): parnn_lowrank_seed. */
int parnn_lowrank_basis(uint64_t dim, uint64_t rank, uint64_t seed, double* out);
uint64_t parnn_lowrank_seed(int layer, int side);
/* allreduce_average on host vectors (parallel.cpp:40-59), fixed midpoint tree */
int parnn_allreduce_average_host(const double* contributions, uint64_t m, uint64_t len, double* out);

/* ---------------- device runtime ---------------------------------------- */
int parnn_ctx_create(int device, parnn_ctx** out);
int parnn_ctx_destroy(parnn_ctx* ctx);
int parnn_ctx_sync(parnn_ctx* ctx);

/* Device-resident Dataset (data.hpp:17-26): features n x d, labels. */
int parnn_dataset_create(parnn_ctx* ctx, const double* x, const int32_t* y, uint64_t n, uint64_t d,
                         uint64_t classes, parnn_dataset** out);
int parnn_dataset_destroy(parnn_dataset* ds);
/* generate_synthetic + split_cv + train-split feature_stats / standardize_in_place
 * (data.cpp:124-242) computed ON THE DEVICE into a train and a CV dataset:
 * labels and row order bit-exact with the reference, features within fp32
 * rounding (the gaussian stream is the reference's Rng(seed) polar-method
 * stream, reconstructed in parallel by xoshiro jump-ahead). */
int parnn_dataset_generate(parnn_ctx* ctx, uint64_t classes, uint64_t dim, uint64_t per_class, double separation,
                           uint64_t seed, double cv_fraction, uint64_t split_seed, int standardize,
                           parnn_dataset** train, parnn_dataset** cv);
/* rows, features, classes of a device dataset */
int parnn_dataset_info(parnn_dataset* ds, uint64_t* n, uint64_t* d, uint64_t* classes);
/* the dataset's fp32 features (n x d row-major) and labels back to the host */
int parnn_dataset_download(parnn_dataset* ds, float* x, int32_t* y);
/* load_csv (data.cpp:66-107): 'label,f1,...' rows, '#' comments, errors with
 * the 1-based line (parsed on all host threads). Buffers of cap_rows x cap_dim;
 * n / d / classes are always set, the arrays only when they fit. */
int parnn_load_csv(const char* path, double* x, int32_t* y, uint64_t cap_rows, uint64_t cap_dim, uint64_t* n,
                   uint64_t* d, uint64_t* classes);
/* load_csv straight into a device dataset */
int parnn_dataset_load_csv(parnn_ctx* ctx, const char* path, parnn_dataset** out);
/* save_csv (data.cpp:109-122): '%.17g' features */
int parnn_save_csv(const char* path, const double* x, const int32_t* y, uint64_t n, uint64_t d);

/* One worker's model + NG state + workspaces (WorkerState, parallel.cpp:81-91). */
int parnn_replica_create(parnn_ctx* ctx, const uint64_t* dims, int ndims, int activation, int precision,
                         int optimizer, uint64_t minibatch, uint64_t max_steps, double ng_decay,
                         double ng_smoothing, parnn_replica** out);
int parnn_replica_destroy(parnn_replica* r);
/* unflatten / flatten (network.cpp:238-272) */
int parnn_replica_set_params(parnn_replica* r, const double* params, uint64_t n);
int parnn_replica_get_params(parnn_replica* r, double* params, uint64_t n);
/* NgState factors: per layer r_in (din^2) then r_out (dout^2) (optimizer.hpp:22-34) */
int parnn_replica_get_ng_state(parnn_replica* r, double* factors, uint64_t n);
int parnn_replica_set_ng_state(parnn_replica* r, const double* factors, uint64_t n, uint64_t update_count);
/* Low-rank NG-SGD knobs (optimizer PARNN_NGSGD_LOWRANK; alpha = ng_smoothing):
 * ranks of the input / output-derivative Fisher factors (<= 96), subspace
 * update period P, initial updates on the first minibatch, the history
 * length S (eta = 1 - exp(-B P / S)) and the update lag (steps until an update
 * takes effect: 1 = the next step; >= 2: computed in the background while the
 * steps in between run; capped at P). Resets the NG state. */
int parnn_replica_set_lowrank(parnn_replica* r, int rank_in, int rank_out, int update_period, int init_iters,
                              double num_samples_history, int update_lag);
/* Low-rank NG state of (layer, side 0 = in [A_prev | 1], 1 = out dz):
 * W = E^1/2 R (rank x dim, row-major), d (rank), rho. */
int parnn_replica_lowrank_state(parnn_replica* r, int layer, int side, double* w, double* d, double* rho,
                                uint64_t* rank, uint64_t* dim);
/* Diagnostics of (layer, side): {tr(X X^T), gamma, Jacobi sweeps, Jacobi SM
 * cycles, eigensolve start, end (%globaltimer ns)} of the last preconditioning
 * / subspace update. */
int parnn_replica_lowrank_diag(parnn_replica* r, int layer, int side, double out[6]);
/* Test hook: one low-rank subspace-update eigensolve (the device kernel of
 * the update) on a given Gram of [J; W] (2R x 2R fp32) and state
 * {d[R], e[R], rho, tr(XX^T), ...} (2R+12 doubles); returns the new state
 * and M (R x 2R, W' = M [J; W]). */
int parnn_debug_lowrank_eig(int rank, uint64_t dim, double eta, double a, double alpha, const double* state_in,
                            const float* gram, double* state_out, float* m_out, int* sweeps);
/* Test hook: ONE production tcgen05 GEMM (the trainer's gemm_plan tile / cluster
 * selection, kernels and fused epilogues) on host fp32 data:
 *   D[m, n] = sum_k A(m, k) B(n, k),  A given as [M x K] (a_mn = 0) or [K x M]
 *   (a_mn = 1), B as [N x K] (b_mn = 0) or [K x N] (b_mn = 1), operands rounded
 *   to the precision's type, fp32 accumulation, then epilogue `mode`
 *   (gemm.cuh EpiMode: 0 act(D + bias[n]), 1 D + bias[n], 2 alpha D,
 *   3 out -= lr alpha D (+ bias column `bias_col` -> bias[m]), 4 D * act'(aux),
 *   5 beta out + alpha D, 6 out += alpha D, 7 out -= D, 8 split-K partials
 *   (summed into out), 9 aux - D (+ sums {aux^2, out^2})).
 * out (M x N) is read for the read-modify-write modes and receives the result;
 * out2 receives the bf16 operand copy (modes 3, 6 in bf16) or the updated bias
 * (mode 3 with bias_col >= 0). force_mc: 0 auto, 1 single-CTA tiles, 2 CTA
 * pairs with 2-SM MMAs, 3 split-K CTA pairs. info[6] = {cluster mode, BN,
 * split-K factor, non-finite flag bits, grid, threads}. */
int parnn_debug_gemm(int precision, int a_mn, int b_mn, int m, int n, int k, int mode, int act, int ksplit,
                     int force_bn, int force_mc, int lower, int bias_col, float alpha, float beta, float lr,
                     const float* a, const float* b, const float* bias, const float* aux, float* out, float* out2,
                     double* sums, int* info);
/* Build the step's GEMM plans + CUDA graph against a training dataset. */
int parnn_replica_bind(parnn_replica* r, parnn_dataset* train);
/* Upload one epoch: steps*minibatch dataset row ids (Dataset::select order) and per-step lr. */
int parnn_replica_upload_epoch(parnn_replica* r, const uint32_t* rows, const float* lrs, uint64_t steps);
/* Enqueue `steps` minibatch updates: forward -> cross_entropy -> backward ->
 * [ng_update_state -> ng_precondition] -> sgd_step_in_place
 * (parallel.cpp:117-130). Asynchronous. */
int parnn_replica_step(parnn_replica* r, uint64_t steps);
/* Wait and raise the reference's errors (cholesky pivot, non-finite gradient). */
int parnn_replica_sync(parnn_replica* r);
/* Per-step batch CE (cross_entropy, network.cpp:145-160) of the current epoch. */
int parnn_replica_ce(parnn_replica* r, double* out, uint64_t steps);
/* Batch CE of step `step` of the current epoch, waiting only for that step
 * (later steps may still run): the pipelined per-step loss readback. */
int parnn_replica_step_ce(parnn_replica* r, uint64_t step, double* out);
/* forward (network.cpp:119-143): last-layer pre-activations for given rows. */
int parnn_replica_forward(parnn_replica* r, parnn_dataset* ds, const uint32_t* rows, uint64_t b, float* z_out);
/* accuracy (network.cpp:274-289) on a whole dataset */
int parnn_replica_accuracy(parnn_replica* r, parnn_dataset* ds, double* acc);
/* number of device kernels one step launches */
int parnn_replica_kernels_per_step(parnn_replica* r, uint64_t* n);
/* Device time (CUDA events on the replica's stream) of `steps` graph launches. */
int parnn_replica_time_steps(parnn_replica* r, uint64_t steps, double* ms);
/* Eager profiled steps: per-region average ms (events between launches on the
 * replica stream) and algorithmic flops; names newline-separated "kind:layer". */
int parnn_replica_profile(parnn_replica* r, uint64_t steps, char* names, uint64_t names_cap, double* ms,
                          double* flops, uint64_t cap, uint64_t* n_regions);
/* Overwrite dataset rows [row0, row0+n) from host fp32 features (+ labels):
 * the per-step host->device input copy of the end-to-end path. */
int parnn_dataset_write_f32(parnn_dataset* ds, const float* x, const int32_t* y, uint64_t row0, uint64_t n);

/* ---------------- averaging / multi-GPU ---------------------------------- */
/* NCCL communicator across processes (one per GPU). */
int parnn_comm_unique_id(unsigned char out[128]);
int parnn_comm_create(parnn_ctx* ctx, const unsigned char id[128], int nranks, int rank, parnn_comm** out);
int parnn_comm_destroy(parnn_comm* c);
/* allreduce_average (parallel.cpp:40-59) over the local replicas (+ comm):
 * every replica is replaced by the mean over m_total workers. */
int parnn_average(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total);
/* A persistent averaging group over the local replicas (+ comm): run() enqueues
 * one averaging event (per-layer buckets, event-gated into each replica's next
 * forward) without blocking the host, as train_parallel's loop does. */
typedef struct parnn_averager parnn_averager;
int parnn_averager_create(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total,
                          parnn_averager** out);
int parnn_averager_run(parnn_averager* a);
int parnn_averager_destroy(parnn_averager* a);
/* Device time (CUDA events on the averaging stream) of `iters` back-to-back
 * averaging events: ms per event, and the fp32 bytes one event reduces per GPU
 * (bus bandwidth = 2 (n-1)/n * bytes / time over n GPUs). */
int parnn_time_average(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total, uint64_t iters,
                       double* ms_per_event, double* bytes);
/* worker_epoch's inner loop (parallel.cpp:106-137) for benchmarking: `steps`
 * minibatch updates on every local replica with an averaging event every
 * avg_frequency updates (and one closing the window); device time in ms. */
int parnn_run_steps(parnn_replica** reps, int n_local, parnn_comm* comm, uint64_t m_total, uint64_t steps,
                    uint64_t avg_frequency, double* ms);

/* ---------------- the train loop ----------------------------------------- */
/* ParallelPlan (parallel.hpp:22-27) + TrainOptions (parallel.hpp:31-38) + placement. */
typedef struct {
    uint64_t workers;        /* m */
    uint64_t avg_frequency;  /* n */
    uint64_t minibatch;      /* B */
    uint64_t base_seed;
    int optimizer;           /* parnn_optimizer */
    int lr_schedule;         /* parnn_lr_variant */
    double lr_init;
    uint64_t epochs;
    double ng_decay;
    double ng_smoothing;
    int precision;           /* parnn_precision */
    int activation;          /* parnn_activation */
    uint64_t rank0;          /* first global rank hosted by this process */
    uint64_t local_workers;  /* ranks hosted here (0 = all m) */
    int serial;              /* serial_train semantics (parallel.cpp:285-294) */
    /* low-rank NG-SGD knobs (PARNN_NGSGD_LOWRANK); 0 = default (20, 80, 4, 2000, lag 4) */
    int ng_rank_in;
    int ng_rank_out;
    int ng_update_period;
    double ng_history;
    int ng_update_lag;       /* 0 = default (4 = the update period) */
} parnn_train_config;

/* train_parallel / serial_train (parallel.cpp:163-294). metrics_out holds up
 * to `epochs` rows of 7 doubles: {epoch, lr, train_ce, cv_accuracy,
 * wall_seconds, workers, avg_events} (EpochMetrics, parallel.hpp:40-48). */
int parnn_train(parnn_ctx* ctx, parnn_comm* comm, const parnn_train_config* cfg, const uint64_t* dims, int ndims,
                const double* params0, parnn_dataset* train, parnn_dataset* cv, double* params_out,
                double* metrics_out, uint64_t* epochs_run);

/* ---------------- RBM CD-1 pretraining (pretrain.hpp) -------------------- */
/* RbmParams packed as [W (h x v) row-major, v_bias (v), h_bias (h)]. */
int parnn_rbm_create(parnn_ctx* ctx, uint64_t visible, uint64_t hidden, int gaussian, uint64_t batch, int precision,
                     parnn_rbm** out);
int parnn_rbm_destroy(parnn_rbm* r);
int parnn_rbm_set_params(parnn_rbm* r, const double* p);
int parnn_rbm_get_params(parnn_rbm* r, double* p);
/* cd1_update (pretrain.cpp:123-125) on `b` rows of a host batch.
 * sampling: 0 counter-based Philox Bernoulli(seed, counter), 1 threshold_half
 * (pretrain.cpp:71-77), 2 host-provided uniforms (u_host, b*h values). */
int parnn_rbm_cd1(parnn_rbm* r, const double* batch, uint64_t b, double lr, int sampling, uint64_t seed,
                  uint64_t counter, const double* u_host);
/* hidden_probs (pretrain.cpp:37-45) for n rows */
int parnn_rbm_hidden_probs(parnn_rbm* r, const double* x, uint64_t n, double* out);
/* reconstruction_error (pretrain.cpp:127-136) */
int parnn_rbm_reconstruction_error(parnn_rbm* r, const double* x, uint64_t n, double* out);
/* greedy_pretrain (pretrain.cpp:162-207): host Rng(seed) drives rbm_init,
 * shuffles and the output-layer init exactly as the reference; Bernoulli
 * draws use the counter-based device RNG (statistical parity only). */
int parnn_greedy_pretrain(parnn_ctx* ctx, const uint64_t* dims, int ndims, const double* data, uint64_t n,
                          uint64_t epochs, double lr_gaussian, double lr_bernoulli, uint64_t batch, uint64_t seed,
                          int precision, double* params_out);

/* greedy_pretrain (pretrain.hpp:74-76) on the CALLER's Rng: rng_state /
 * rng_spare / rng_has_spare hold the xoshiro256** state words and the polar
 * gaussian cache of the caller's parnn::Rng (rng.hpp) and are updated in place
 * to the state the reference leaves (rbm_init, per-epoch shuffles and the
 * Bernoulli draws consumed exactly as pretrain.cpp:162-207 does; the output
 * layer's Glorot init is bit-identical). `activation` is the model's
 * (network.hpp:16); RBM layers are sigmoid as in the reference. */
int parnn_greedy_pretrain_rng(parnn_ctx* ctx, const uint64_t* dims, int ndims, const double* data, uint64_t n,
                              uint64_t epochs, double lr_gaussian, double lr_bernoulli, uint64_t batch,
                              int activation, uint64_t rng_state[4], double* rng_spare, int* rng_has_spare,
                              int precision, double* params_out);

/* Device time (CUDA events around each layer's epoch loop) of the CD-1 steps
 * of the last greedy_pretrain call on this thread, their count and their flop
 * (10 v h b per step). Measurement aid: the reference has no counterpart. */
int parnn_pretrain_last_stats(double* cd1_device_seconds, uint64_t* cd1_steps, double* cd1_flop);

#ifdef __cplusplus
}
#endif
#endif
