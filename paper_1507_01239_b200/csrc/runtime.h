// Device runtime of the B200 trainer: contexts, device-resident datasets,
// replicas (one model + NG state + workspaces on one GPU) and the fused
// per-minibatch step. Everything here is C++; the C ABI (capi.cpp) wraps it.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gemm.cuh"

#define CUDA_THROW(x)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                                     __FILE__ + ":" + std::to_string(__LINE__) + ")");             \
    } while (0)

namespace pnb {

using bf16 = __nv_bfloat16;

// Blocking host -> device upload. cudaMemcpy from pageable memory may return
// before its DMA has landed, and the legacy stream it runs on does not order
// the non-blocking streams every kernel here is launched on: wait for it.
inline void upload(void* dst, const void* src, size_t bytes) {
    CUDA_THROW(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    CUDA_THROW(cudaStreamSynchronize(cudaStreamLegacy));
}
// Blocking zero fill (cudaMemset is asynchronous on the legacy stream; same hazard).
inline void zero(void* dst, size_t bytes) {
    CUDA_THROW(cudaMemset(dst, 0, bytes));
    CUDA_THROW(cudaStreamSynchronize(cudaStreamLegacy));
}

struct GemmPlan {
    CUtensorMap ta, tb;
    dim3 grid;
    int smem = 0, M = 0, N = 0, K = 0, bn = 0, threads = 128, tiles = 0;
    int mc = 1;  // 2: CTA pairs (clusters of 2) computing 256 x BN tiles with 2-SM MMAs
    int prec = 0;
    bool a_mn = false, b_mn = false;
    GemmEpi ep;
    void* fn = nullptr;
};

// One persistent launch over the problems of several plans -- the step's dW
// GEMMs (gemm.cuh, NP > 1). Every member: bf16 operands, both MN-major, BN =
// 256, transposed-epilogue mode, single-CTA tiles, no split-K.
struct GemmGroupPlan {
    GemmParams<kGroupMax> args;
    dim3 grid;
    int smem = 0, threads = 320, tiles = 0, np = 0;
    void* fn = nullptr;
};
bool gemm_groupable(const GemmPlan& p);
void gemm_group_plan(GemmGroupPlan& g, const std::vector<const GemmPlan*>& parts, int num_sms);
void gemm_group_launch(const GemmGroupPlan& g, cudaStream_t s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// function attributes are per device and the C ABI allows contexts on several
// devices (and replicas built from several threads) in one process.
void ensure_smem_attr(const void* fn, int bytes);

int choose_bn(int M, int N, int num_sms);
// prec: 0 = BF16 operands, 1 = TF32, 2 = fp32 via 3xTF32 split
// force_mc (tests / tuning): 0 = automatic, 1 = single-CTA tiles, 2 = CTA pairs
// with 2-SM MMAs, 3 = split-K CTA pairs (bf16 only for 2 and 3)
void gemm_plan(GemmPlan& p, int prec, bool a_mn, const void* A, long lda, bool b_mn, const void* B, long ldb,
               int M, int N, int K, const GemmEpi& ep, int num_sms, int force_bn = 0, int force_mc = 0);
void gemm_launch(const GemmPlan& p, cudaStream_t s);
// Cap on the persistent grid of subsequent launches from this thread (0 = none):
// steps that run long single-CTA kernels (the NG subspace eigensolves) beside
// the GEMMs keep those SMs out of the GEMM grids, so no GEMM CTA waits for them.
void gemm_set_grid_cap(int cap);
// PDL on / off for the GEMMs this thread launches next (default on)
void gemm_set_pdl(bool on);
dim3 gemm_launch_grid(const GemmPlan& p);

enum Precision : int { PREC_BF16 = 0, PREC_TF32 = 1, PREC_FP32 = 2 };
enum Optimizer : int { OPT_SGD = 0, OPT_NG_KRON = 1, OPT_NG_LOWRANK = 2 };

inline long pad32(long v) { return (v + 31) / 32 * 32; }

struct Context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t avg = nullptr;  // model averaging (parallel.cu Averager), apart from host copies
    explicit Context(int dev);
    ~Context();
};

struct DeviceDataset {
    Context* ctx;
    long n = 0, d = 0, ld = 0, classes = 0;
    float* x32 = nullptr;  // [n x ld] fp32 (zero padded)
    bf16* x16 = nullptr;   // [n x ld] bf16 copy, created on first bf16 use
    int32_t* y = nullptr;
    cudaEvent_t written = nullptr;  // last write_rows; steps of replicas bound here wait on it
    DeviceDataset(Context* c, const double* x, const int32_t* labels, long n, long d, long classes);
    DeviceDataset(Context* c, long n, long d, long classes);  // zeroed device buffers (data.cu fills them)
    ~DeviceDataset();
    const void* features(Precision p);
    // overwrite rows [row0, row0+n) from host fp32 (+ labels); refreshes the bf16 copy
    void write_rows(const float* x, const int32_t* y, long row0, long n, cudaStream_t s);
};

// Host-visible error record written by device kernels (pivot failures).
struct DevErr {
    int chol_failed;  // 1 if any Cholesky pivot failed
    int chol_index;
    float chol_value;
    int pad;
};

// Smoothed Kronecker factor S = R + lambda I, factored in place by the blocked
// Cholesky of ng.cu (128-row blocks; diagonal blocks on SIMT, panel and
// trailing updates as 3xTF32 tcgen05 GEMMs).
constexpr int NG_NB = 128;
struct NgFactor {
    long n = 0, ld = 0;
    float* a = nullptr;     // [n x ld]: S, overwritten by L (lower triangle)
    float* linv = nullptr;  // [nblk x NB x NB]: inverses of the diagonal blocks of L
    std::vector<GemmPlan> panel, col, rest;  // per block: panel solve, look-ahead column, rest of trailing
    cudaStream_t fs = nullptr, ts = nullptr;  // critical-path / bulk-trailing streams
    std::vector<cudaEvent_t> ev_panel, ev_trail;
};
struct NgSolve {  // X <- S^-1 X for one fixed right-hand-side buffer
    std::vector<GemmPlan> fdiag, fupd, bdiag, bupd;  // per block
    // backward sweep in block pairs (i, i-1): X_{i-1} -= L_{i,i-1}^T X_i (bnext), then
    // X_{<i-1} -= L_{{i-1,i},<i-1}^T X_{i-1,i} with K = 256 (bpair); indexed by i
    std::vector<GemmPlan> bnext, bpair;
    // forward sweep in block pairs (i, i+1): X_{i+1} -= L_{i+1,i} X_i (fnext), then
    // X_{>i+1} -= L_{>i+1,{i,i+1}} X_{i,i+1} with K = 256 (fpair); indexed by i
    std::vector<GemmPlan> fnext, fpair;
};
struct NgLayer {
    NgFactor out, in;
    NgSolve solve_out, solve_in;
    float* t1 = nullptr;  // [dout x ldt]: [G | g_b], solved in place by S_out
    float* t2 = nullptr;  // [din x ld2]: (S_out^-1 G)^T, solved in place by S_in
    long ldt = 0, ld2 = 0;
    double* part = nullptr;         // norm-reduction scratch
    cudaStream_t stream = nullptr;  // the layer's NG chain runs concurrently with the others
    cudaEvent_t done = nullptr, ev_ready = nullptr, ev_in_done = nullptr;
};

// NG-SGD low-rank online preconditioner (ng_lowrank.cu; SURVEY §8a A17,
// Povey et al. 2014). One side = one of the two per-example vector sets of a
// layer: "in" = [A_prev | 1] (D = din + 1), "out" = dz (D = dout).
constexpr int LR_MAX_RANK = 96;
struct LrConfig {
    int rank_in = 20, rank_out = 80;  // Kaldi nnet2/3 defaults
    int update_period = 4;            // subspace update every P minibatches
    int init_iters = 3;               // updates on the first minibatch before use
    double history = 2000.0;          // S: eta = 1 - exp(-B P / S)
    int update_lag = 4;               // steps until an update takes effect (1 = next step; <= P)
    double alpha = 4.0;               // smoothing (the reference's ng_smoothing)
};
struct LrSide {
    bool in = false;
    long dx = 0;  // columns of X proper (din or dout)
    long D = 0;   // dx (+1 for the ones column)
    int R = 0;
    int ns = 1;  // W operand rows per direction: 1 (fp32 modes), 2 (bf16: W_hi, W_lo)
    long ldY = 0, ldH = 0, ldx = 0, ldxh = 0;  // ldx: X's rows; ldxh: xhat's (in side: + the ones column)
    float* YW = nullptr;    // [2R x ldY] fp32: rows [0,R) J = H^T X, rows [R,2R) W (master)
    void* wop = nullptr;    // bf16 operand copy [W_hi; W_lo] [2R x ldY] (fp32 modes: the W rows of YW)
    float* hpart = nullptr; // [S x B x ns*R] split-K partials of H = X W^T
    void* H = nullptr;      // [B x ldH] operand-typed H (bf16: [H | H])
    float* ohat = nullptr;  // [B] preconditioned ones column (in side)
    double* rpart = nullptr;  // [nrb x (R+1)]: per-CTA column sums of H, sum of ohat^2
    double* xpart = nullptr;  // [grid x 2]: per-CTA sums of X^2 and Xhat^2
    float* gpart = nullptr;   // [S2 x 2R x 2R] Gram partials of [J; W]
    float* gram = nullptr;    // [2R x 2R]
    double* st = nullptr;     // d[R], e[R], rho, tr(X X^T), gamma, diagnostics
    double* stn = nullptr;    // the computed update's state (committed over st)
    double* trxx_snap = nullptr;  // tr(X X^T) of the step the update is computed from
    float* Wn = nullptr;      // [R x ldY] the computed update's W
    void* wopn = nullptr;     // its bf16 [W_hi; W_lo] (bf16 mode)
    float* M = nullptr;       // [R x 2R]: W' = M [J; W]
    void* xhat = nullptr;     // [B x ldxh] preconditioned vectors (operand dtype); in side: column dx = ohat
    const void* X = nullptr;  // [B x ldx] the layer's vectors (acts[l] or dz[l])
    GemmPlan hg, xg, jg, gg;
    int nrb = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
};
enum LrVariantBits : int {
    LRV_INIT = 1,      // first step: init updates on its own batch
    LRV_J = 2,         // compute J of an update at the end of the step
    LRV_APPLY = 4,     // lag 1: compute + commit the pending update at the start of the step
    LRV_COMMIT = 8,    // lag >= 2: commit the update computed in the background
    LRV_INFLIGHT = 16,  // lag >= 2: the background update runs beside this step (GEMM grids capped)
    // averaging gates (every optimizer): captured only into the steps that need them
    GATE_WAIT = 32,  // an average is pending: wait on ev_gate[l] before the forward GEMM of layer l
    GATE_REC = 64,   // the step ends an averaging window: record ev_upd[l] once layer l is final
    kVariants = 128
};
struct LrLayer {
    LrSide in, out;
    float* coef = nullptr;  // gamma_in * gamma_out (device)
};

struct Profile {
    std::vector<cudaEvent_t> events;
    std::vector<std::string> names;
    std::vector<double> flops;
};

struct Replica {
    Context* ctx;
    cudaStream_t stream = nullptr;  // private stream: local replicas step concurrently
    cudaStream_t side = nullptr;    // dW GEMMs, concurrent with the dA chain
    std::vector<cudaEvent_t> ev_bwd, ev_dw;
    cudaEvent_t ev_side = nullptr;
    std::vector<long> dims;  // input, hidden..., output
    int L = 0;
    int act = 0;
    Precision prec = PREC_BF16;
    Optimizer opt = OPT_SGD;
    long B = 0;  // minibatch (fixed per replica)
    long max_steps = 0;
    double ng_decay = 0.95, ng_smoothing = 4.0;
    long ng_t = 0;  // EMA update count (same for every layer)

    // padded flat parameter layout: per layer W [dout x ldw] then b [pad32(dout)]
    std::vector<long> ldw, w_off, b_off;
    long n_pad = 0;  // floats in the padded parameter buffer
    float* params = nullptr;
    bf16* wshadow = nullptr;  // bf16 operand copy of the weights (bf16 mode), same offsets
    float* grads = nullptr;   // padded fp32 gradients (NG mode: G then preconditioned)

    // activations: act[0] = gathered input batch; act[l+1] = output of layer l (hidden only)
    std::vector<void*> acts;
    std::vector<long> ld_act;
    float* zout = nullptr;  // last layer pre-activation [B x ld_act[L]]
    std::vector<void*> dz;  // per layer [B x ld_act[l+1]] (op dtype)
    std::vector<float*> r_in, r_out;  // NG factors [n x pad32(n)]
    std::vector<NgLayer> ngl;         // per-layer Cholesky/TRSM workspaces and GEMM plans
    cudaEvent_t ng_fork = nullptr;
    double* scal = nullptr;   // per-layer scalars: traces, norms (device)

    // per-epoch device state
    int* d_step = nullptr;
    float* d_lr = nullptr;        // [max_steps]
    uint32_t* d_rows = nullptr;   // [max_steps * B] dataset row ids
    int32_t* d_ybatch = nullptr;  // [B]
    float* ce_rows = nullptr;     // [B]
    double* d_ce = nullptr;       // [max_steps] batch-mean CE
    unsigned* d_flags = nullptr;  // non-finite weight/bias grad bits (2 per layer)
    DevErr* d_err = nullptr;
    // accuracy(): row ids of the evaluated set and the correct counter, kept
    // across calls (zeroed on the replica stream, not by a legacy-stream memset)
    uint32_t* eval_rows = nullptr;
    long eval_rows_n = 0;
    unsigned long long* eval_correct = nullptr;

    // Per-layer averaging buckets (parallel.cu Averager). ev_upd[l] is recorded
    // inside every step (graph: external record node) once layer l's update is
    // final; the averager waits on it, averages layer l's [W_l | b_l] range on
    // its own stream and records ev_gate[l]; every step waits on ev_gate[l]
    // (graph: external wait node) right before its forward GEMM of layer l. So
    // the average of the last layers overlaps the next step's first layers.
    std::vector<cudaEvent_t> ev_upd, ev_gate;
    cudaEvent_t ev_tail = nullptr;  // end of the last step (averaging after a step launched without GATE_REC)
    bool gate_pending = false;      // an average was enqueued: the next step waits on the gates
    bool last_recorded = false;     // the last step recorded ev_upd (GATE_REC)
    long bucket_begin(int l) const { return w_off[l]; }
    long bucket_end(int l) const { return l + 1 < L ? w_off[l + 1] : n_pad; }

    DeviceDataset* bound = nullptr;  // dataset the plans/graph were built for
    std::vector<GemmPlan> fwd, dw, da, mom_in, mom_out;
    // every layer's dW GEMM (+ SGD update) in one persistent grouped launch
    // (bf16 SGD and low-rank NG; PARNN_NO_DW_GROUP=1 launches them per layer)
    GemmGroupPlan dwg;
    bool dw_group = false;
    // bf16 SGD: every activation buffer feeding a dW GEMM carries a constant-1
    // column at index d_l, so the GEMM's extra output column is the bias
    // gradient (sum over the batch of dz, network.cpp:203-208) and the epilogue
    // updates the bias with the weights -- no separate bias-gradient kernel
    bool bias_in_dw = false;
    long ones_col0() const { return bias_in_dw ? dims[0] : -1; }
    cudaGraphExec_t graph = nullptr;  // the plain step (SGD / kron-full): alias of vgraphs[0]
    bool use_graph = true;
    long kernels_per_step = 0;

    // NG low-rank (OPT_NG_LOWRANK): per-layer state, the host step counter
    // that selects the graph variant (init / Fisher-update / plain), one
    // captured graph per variant
    LrConfig lrc;
    std::vector<LrLayer> lrl;
    long lr_t = 0;
    int variant = 0;  // LRV_* bits of the current step
    std::vector<cudaGraphExec_t> vgraphs;
    std::vector<long> vnodes;
    std::vector<cudaEvent_t> ev_act;  // acts[l] ready (in-side chains start)
    cudaEvent_t ev_t0 = nullptr;
    int lr_variant(long t) const;
    int lr_lag() const;
    // lag-2 updates: computed by a separate graph on `bg` while the next step runs
    cudaStream_t bg = nullptr;
    cudaGraphExec_t apply_graph = nullptr;
    cudaEvent_t ev_jdone = nullptr, ev_applied = nullptr;
    bool apply_pending = false;
    long apply_nodes = 0;
    void capture_variant(int v);
    // capture the averaging-gated variants of every step kind up front (an averaging
    // group does this, so no capture happens inside a timed or steady-state loop)
    void precapture_gates();
    void capture_apply_graph();
    void lr_before_step(cudaStream_t s);
    void lr_after_step(cudaStream_t s);
    void set_lowrank(const LrConfig& c);
    void get_lowrank_state(int layer, int side, double* w, double* d, double* rho) const;

    Replica(Context* c, const std::vector<long>& dims, int act, Precision p, Optimizer o, long batch,
            long max_steps, double decay, double smoothing);
    ~Replica();

    bool f32() const { return prec != PREC_BF16; }  // fp32 storage of operands
    size_t esz() const { return f32() ? 4 : 2; }
    void set_params(const double* flat);  // canonical flatten order (network.cpp:238-248)
    void get_params(double* flat) const;
    void set_ng_state(const double* factors, long t);
    void get_ng_state(double* factors) const;

    void bind(DeviceDataset* ds);  // build GEMM plans + graph for this dataset
    void upload_epoch(const uint32_t* rows, const float* lrs, long steps);
    // per-step completion events (ring): the loss of step j of the epoch can be
    // read while later steps run (pipelined end-to-end loop)
    static constexpr int kStepRing = 64;
    std::vector<cudaEvent_t> step_ev;
    long epoch_steps = 0;  // steps launched since upload_epoch
    long epoch_len = 0;    // steps uploaded
    double step_ce(long j);
    // one minibatch (graph or eager); window_end: an average follows this step
    void run_step(cudaStream_t s, bool window_end = false);
    void enqueue_step(cudaStream_t s);
    void sync_shadow(cudaStream_t s);  // recompute bf16 copy after external param writes
    void check_errors();               // throws the reference's messages

    // optional timeline of the concurrent step (PARNN_TIMELINE=1): timing events
    // captured into the graph, dumped to stderr by check_errors()
    std::vector<std::pair<std::string, cudaEvent_t>> tl;
    std::vector<cudaEvent_t> tl_pool;
    void tmark(const std::string& name, cudaStream_t s);
    void dump_timeline();

    // live per-region timing with CUDA events on the replica stream (bench)
    Profile* prof = nullptr;
    void mark(const char* kind, int layer, double flops, cudaStream_t s);
    void profile_steps(long steps, std::vector<std::string>& names, std::vector<double>& ms,
                       std::vector<double>& flops);
    double time_steps(long steps);  // ms for `steps` graph launches (CUDA events)

    // debug/test hooks
    void forward_only(DeviceDataset* ds, const uint32_t* rows, long b, float* zout_host);
    double accuracy(DeviceDataset* ds);
};

void debug_gemm(int prec, bool a_mn, bool b_mn, int M, int N, int K, int mode, int act, int ksplit, int force_bn,
                int force_mc, int lower, int bias_col, float alpha, float beta, float lr, const float* a,
                const float* b, const float* bias, const float* aux, float* out, float* out2, double* sums,
                int* info);
// non-blocking stream at priority level 0 (highest: the dz chain and whatever
// gates it), 1 (concurrent side work) or 2 (lowest: background NG subspace updates)
cudaStream_t make_stream(int level);
// data.cu: generate_synthetic + split_cv + train-split standardize (data.cpp:124-242)
// on the device; labels / row order bit-exact, features within fp32 rounding
void generate_device(Context* ctx, uint64_t classes, uint64_t dim, uint64_t per_class, double sep, uint64_t seed,
                     double cv_fraction, uint64_t split_seed, bool standardize, DeviceDataset** train,
                     DeviceDataset** cv);
void record_ext(cudaEvent_t e, cudaStream_t s);
void wait_ext(cudaStream_t s, cudaEvent_t e);

// ----------------------------------------------------------- kernels.cu
void launch_gather(const void* x, long ldx, const int32_t* y, const uint32_t* rows, const int* step, long B,
                   long d, void* out, long ldo, int32_t* yout, bool f32, cudaStream_t s, long ones_col = -1);
void launch_fill_ones_column(void* buf, long ld, long rows, long col, bool f32, cudaStream_t s);
void launch_softmax_ce(const float* z, long ldz, long B, long C, const int32_t* y, void* dz, long lddz,
                       float* ce_rows, bool f32, cudaStream_t s);
void launch_ce_reduce(const float* ce_rows, long B, double* d_ce, int* step, int advance, cudaStream_t s);
void launch_bias_grad(const void* dz, long lddz, long B, long C, bool f32, float* bias, float* gb, const float* lr,
                      const int* step, unsigned* flags, unsigned bit, cudaStream_t s);
void launch_f32_to_bf16_rows(const float* src, long ld, long rows, long cols, bf16* dst, cudaStream_t s);
void launch_convert_dataset(const float* x32, long n, long ld, bf16* x16, cudaStream_t s);
void launch_argmax_correct(const float* z, long ldz, long B, long C, const int32_t* y, unsigned long long* correct,
                           cudaStream_t s);

// NG kron-full (ng.cu)
void ng_alloc(Replica& r);
void ng_free(Replica& r);
void ng_build_plans(Replica& r);
void ng_precondition_layer(Replica& r, int l, cudaStream_t s);
void ng_apply_update(Replica& r, int l, cudaStream_t s);

// NG low-rank (ng_lowrank.cu)
void lr_alloc(Replica& r);
void lr_free(Replica& r);
void lr_build_plans(Replica& r);
void lr_precondition_side(Replica& r, LrSide& sd, cudaStream_t s);  // H, Xhat, gamma
void lr_start_update(Replica& r, LrSide& sd, cudaStream_t s);       // J = H^T X
void lr_apply_update(Replica& r, LrSide& sd, cudaStream_t s);       // Gram, eig, W' (into next buffers)
void lr_commit_update(Replica& r, LrSide& sd, cudaStream_t s);      // next buffers -> current
void lr_layer_update(Replica& r, int l, cudaStream_t s);            // bias + dW with gamma
void lr_debug_eig(int R, long D, double eta, double a, double alpha, const double* st_in, const float* gram,
                  double* st_out, float* m_out, int* sweeps);

}  // namespace pnb
