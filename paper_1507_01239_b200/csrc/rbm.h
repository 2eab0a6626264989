// RBM CD-1 pretraining on device (pretrain.hpp / pretrain.cpp).
#pragma once
#include <vector>

#include "host.h"
#include "runtime.h"

namespace pnb {

struct RbmDevice {
    Context* ctx;
    cudaStream_t stream = nullptr;
    long v, h, B;
    bool gaussian;
    Precision prec;
    long ldv, ldh;
    float* W = nullptr;  // [h x ldv] fp32 master
    bf16* Ws = nullptr;  // bf16 operand copy
    float* vb = nullptr;
    float* hb = nullptr;
    void* XR = nullptr;  // [2B x ldv] op dtype: batch rows, then reconstruction rows (= XRs[slot])
    void* XRs[2] = {nullptr, nullptr};  // two buffers: the next batch gathers while a step runs
    void* PN = nullptr;  // [2B x ldh] op dtype: pos probs, then -neg probs
    void* HS = nullptr;  // [B x ldh] op dtype: hidden samples
    double* u_dev = nullptr;  // injected uniforms [B x h]
    double* red = nullptr;    // reduction scratch
    float* part = nullptr;    // split-K partial tiles of the M = b GEMMs
    size_t part_n = 0;
    double* colp = nullptr;   // per-row-chunk column sums: pos - neg [ch_h x ldh], v - recon [ch_v x ldv]
    float* ZP = nullptr;      // [B x ldh] pre-activations of the pos pass (for the fp64 pos - neg)
    uint64_t* dctr = nullptr; // {step, Philox counter base} of graph-launched CD-1 steps
    int ch_h = 1, ch_v = 1;   // row chunks (grid.y) of the h- and v-wide reductions
    long planned_b = -1;
    GemmPlan g_pos, g_recon, g_neg, g_upd;  // the current buffer's plans
    GemmPlan slot_plans[2][4];
    // graph capture only: the bias update on this stream beside the weight update
    cudaStream_t bias_side = nullptr;
    cudaEvent_t ev_neg = nullptr, ev_bias = nullptr;
    bool bias_pending = false;

    RbmDevice(Context* c, long visible, long hidden, bool gaussian, long batch, Precision p);
    ~RbmDevice();
    bool f32() const { return prec != PREC_BF16; }
    void set_params(const double* p);  // [W, v_bias, h_bias]
    void get_params(double* p);
    void plan(long b);
    void use_slot(int sl);  // XR and the plans of buffer sl
    // one CD-1 update on the b rows already in XR[0:b)
    void cd1(long b, double lr, int sampling, uint64_t seed, uint64_t counter);
    void cd1_host(const double* batch, long b, double lr, int sampling, uint64_t seed, uint64_t counter,
                  const double* u);
    // hidden probabilities of the first `rows` rows in XR -> out32 (fp32, ld32)
    void hidden_probs_rows(long rows, float* out32, long ld32);
    void hidden_probs_host(const double* x, long n, double* out);
    double reconstruction_error_host(const double* x, long n);
};

// Device time of the last greedy_pretrain's CD-1 epochs on this thread (events
// around each layer's epoch loop), its step count and 10 v h b flop per step.
struct PretrainStats {
    double cd1_seconds = 0.0;
    uint64_t cd1_steps = 0;
    double cd1_flop = 0.0;
};
extern thread_local PretrainStats g_pretrain_stats;

// rng: the caller's generator, advanced exactly as the reference advances it;
// philox_seed keys the device Bernoulli draws.
void greedy_pretrain(Context* ctx, const std::vector<long>& dims, const double* data, long n, uint64_t epochs,
                     double lr_g, double lr_b, long batch, host::Rng& rng, uint64_t philox_seed, Precision prec,
                     double* params_out);

}  // namespace pnb
