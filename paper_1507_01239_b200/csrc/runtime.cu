// Contexts, device-resident datasets and replicas; the fused minibatch step
// (worker_epoch's body, parallel.cpp:117-130) as one CUDA graph.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "runtime.h"

namespace pnb {

namespace {

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CUDA_THROW(cudaMalloc(&p, n * sizeof(T)));
    zero(p, n * sizeof(T));
    return static_cast<T*>(p);
}

void dfree(void* p) {
    if (p) cudaFree(p);
}

// EMA coefficients of ema_update (optimizer.cpp:64-75) for t = ++(*t_dev):
// coef = {keep, add / B}; t == 1 assigns the batch moment.
__global__ void ng_coeff_kernel(long* t_dev, double rho, double inv_b, float* coef) {
    const long t = *t_dev + 1;
    *t_dev = t;
    double keep = 0.0, add = 1.0;
    if (t > 1) {
        const double denom = 1.0 - pow(rho, (double)t);
        keep = rho * (1.0 - pow(rho, (double)(t - 1))) / denom;
        add = (1.0 - rho) / denom;
    }
    coef[0] = (float)keep;
    coef[1] = (float)(add * inv_b);
}

// Record the first step whose gradients were non-finite, then clear the
// per-step bits (so the host can name the layer the reference would).
__global__ void flags_latch_kernel(unsigned* flags, const int* step) {
    if (flags[0] && !flags[1]) {
        flags[1] = flags[0];
        flags[2] = (unsigned)*step;
    }
    flags[0] = 0;
}

// ... and the step's end: the device step counter advances (the loss was reduced beside the step)
__global__ void flags_latch_advance_kernel(unsigned* flags, int* step) {
    if (flags[0] && !flags[1]) {
        flags[1] = flags[0];
        flags[2] = (unsigned)*step;
    }
    flags[0] = 0;
    *step += 1;
}

}  // namespace

// Event record / wait that become external event nodes when the stream is
// being captured into a graph (a plain record inside a capture is only a
// fork/join marker), so they synchronise with work outside the graph.
void record_ext(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs;
    CUDA_THROW(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        CUDA_THROW(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else
        CUDA_THROW(cudaEventRecord(e, s));
}

cudaStream_t make_stream(int level) {
    int least = 0, greatest = 0;
    CUDA_THROW(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    const int prio = level <= 0 ? greatest : (level >= 2 ? least : (least + greatest) / 2);
    cudaStream_t s;
    CUDA_THROW(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
    return s;
}

// Kernel nodes of a captured graph (event record / wait and memcpy nodes are not kernels).
long count_kernel_nodes(cudaGraph_t g) {
    size_t n = 0;
    CUDA_THROW(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CUDA_THROW(cudaGraphGetNodes(g, nodes.data(), &n));
    long k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        CUDA_THROW(cudaGraphNodeGetType(nd, &t));
        k += t == cudaGraphNodeTypeKernel;
    }
    return k;
}

void wait_ext(cudaStream_t s, cudaEvent_t e) {
    cudaStreamCaptureStatus cs;
    CUDA_THROW(cudaStreamIsCapturing(s, &cs));
    CUDA_THROW(cudaStreamWaitEvent(s, e, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
}

Context::Context(int dev) : device(dev) {
    CUDA_THROW(cudaSetDevice(dev));
    CUDA_THROW(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_THROW(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    avg = make_stream(0);  // the next steps' forwards wait on its gates
}

Context::~Context() {
    if (stream) cudaStreamDestroy(stream);
    if (avg) cudaStreamDestroy(avg);
}

DeviceDataset::DeviceDataset(Context* c, const double* x, const int32_t* labels, long n_, long d_, long classes_)
    : ctx(c), n(n_), d(d_), ld(pad32(d_)), classes(classes_) {
    CUDA_THROW(cudaSetDevice(c->device));
    std::vector<float> h(static_cast<size_t>(n * ld), 0.f);
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < d; ++j) h[i * ld + j] = static_cast<float>(x[i * d + j]);
    for (long i = 0; i < n; ++i)
        if (labels[i] < 0 || labels[i] >= classes)
            throw std::runtime_error("dataset: label " + std::to_string(labels[i]) + " at row " + std::to_string(i) +
                                     " out of range [0, " + std::to_string(classes) + ")");
    x32 = dalloc<float>(h.size());
    y = dalloc<int32_t>(n);
    upload(x32, h.data(), h.size() * 4);
    upload(y, labels, n * 4);
}

DeviceDataset::DeviceDataset(Context* c, long n_, long d_, long classes_)
    : ctx(c), n(n_), d(d_), ld(pad32(d_)), classes(classes_) {
    CUDA_THROW(cudaSetDevice(c->device));
    x32 = dalloc<float>(static_cast<size_t>(n * ld));
    y = dalloc<int32_t>(n);
}

DeviceDataset::~DeviceDataset() {
    if (written) cudaEventDestroy(written);
    dfree(x32);
    dfree(x16);
    dfree(y);
}

const void* DeviceDataset::features(Precision p) {
    if (p != PREC_BF16) return x32;
    if (!x16) {
        x16 = dalloc<bf16>(static_cast<size_t>(n * ld));
        launch_convert_dataset(x32, n, ld, x16, ctx->stream);
        CUDA_THROW(cudaStreamSynchronize(ctx->stream));
    }
    return x16;
}

void DeviceDataset::write_rows(const float* x, const int32_t* labels, long row0, long cnt, cudaStream_t s) {
    if (row0 < 0 || row0 + cnt > n) throw std::runtime_error("dataset: write beyond the dataset");
    CUDA_THROW(cudaMemcpy2DAsync(x32 + row0 * ld, ld * 4, x, d * 4, d * 4, cnt, cudaMemcpyHostToDevice, s));
    if (labels) CUDA_THROW(cudaMemcpyAsync(y + row0, labels, cnt * 4, cudaMemcpyHostToDevice, s));
    if (x16) launch_f32_to_bf16_rows(x32 + row0 * ld, ld, cnt, ld, x16 + row0 * ld, s);
    if (!written) CUDA_THROW(cudaEventCreateWithFlags(&written, cudaEventDisableTiming));
    CUDA_THROW(cudaEventRecord(written, s));
}

Replica::Replica(Context* c, const std::vector<long>& dims_, int act_, Precision p, Optimizer o, long batch,
                 long max_steps_, double decay, double smoothing)
    : ctx(c), dims(dims_), act(act_), prec(p), opt(o), B(batch), max_steps(max_steps_), ng_decay(decay),
      ng_smoothing(smoothing) {
    if (dims.size() < 2) throw std::runtime_error("replica: need at least 2 dims");
    for (long d : dims)
        if (d <= 0) throw std::runtime_error("replica: zero layer dimension");
    if (B <= 0) throw std::runtime_error("replica: minibatch must be >= 1");
    CUDA_THROW(cudaSetDevice(c->device));
    stream = make_stream(0);  // the forward / dz chain: the step's critical path
    side = make_stream(1);
    CUDA_THROW(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
    L = static_cast<int>(dims.size()) - 1;
    ev_bwd.resize(L);
    ev_dw.resize(L);
    ev_upd.resize(L);
    ev_gate.resize(L);
    for (int l = 0; l < L; ++l) {
        CUDA_THROW(cudaEventCreateWithFlags(&ev_bwd[l], cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&ev_dw[l], cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&ev_upd[l], cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&ev_gate[l], cudaEventDisableTiming));
    }
    CUDA_THROW(cudaEventCreateWithFlags(&ev_tail, cudaEventDisableTiming));
    long off = 0;
    for (int l = 0; l < L; ++l) {
        ldw.push_back(pad32(dims[l]));
        w_off.push_back(off);
        off += dims[l + 1] * ldw[l];
        b_off.push_back(off);
        off += pad32(dims[l + 1]);
    }
    n_pad = off;
    params = dalloc<float>(n_pad);
    if (!f32()) wshadow = dalloc<bf16>(n_pad);
    if (opt == OPT_NG_KRON) grads = dalloc<float>(n_pad);
    if (opt == OPT_NG_LOWRANK) lrc.alpha = ng_smoothing;
    bias_in_dw = !f32() && opt == OPT_SGD;
    for (int l = 0; l <= L; ++l) ld_act.push_back(pad32(dims[l] + (bias_in_dw && l < L ? 1 : 0)));
    for (int l = 0; l < L; ++l) acts.push_back(f32() ? (void*)dalloc<float>(B * ld_act[l]) : (void*)dalloc<bf16>(B * ld_act[l]));
    if (bias_in_dw) {  // the constant-1 column of every layer input (acts[0]'s is set by each gather)
        for (int l = 1; l < L; ++l) launch_fill_ones_column(acts[l], ld_act[l], B, dims[l], false, stream);
        CUDA_THROW(cudaStreamSynchronize(stream));
    }
    acts.push_back(nullptr);  // the last layer keeps Z (fp32) in zout
    zout = dalloc<float>(B * ld_act[L]);
    for (int l = 0; l < L; ++l)
        dz.push_back(f32() ? (void*)dalloc<float>(B * ld_act[l + 1]) : (void*)dalloc<bf16>(B * ld_act[l + 1]));
    if (opt == OPT_NG_KRON) {
        for (int l = 0; l < L; ++l) {
            r_in.push_back(dalloc<float>(dims[l] * pad32(dims[l])));
            r_out.push_back(dalloc<float>(dims[l + 1] * pad32(dims[l + 1])));
        }
        ng_alloc(*this);
    }
    if (opt == OPT_NG_LOWRANK) {
        lr_alloc(*this);
        ev_act.resize(L);
        for (auto& e : ev_act) CUDA_THROW(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&ev_t0, cudaEventDisableTiming));
    }
    scal = dalloc<double>(16 * (L + 1) + 512);
    d_step = dalloc<int>(4);
    d_lr = dalloc<float>(std::max<long>(max_steps, 1));
    d_rows = dalloc<uint32_t>(std::max<long>(max_steps, 1) * B);
    d_ybatch = dalloc<int32_t>(B);
    ce_rows = dalloc<float>(B);
    d_ce = dalloc<double>(std::max<long>(max_steps, 1));
    d_flags = dalloc<unsigned>(4);
    d_err = dalloc<DevErr>(1);
}

Replica::~Replica() {
    if (stream) cudaStreamSynchronize(stream);
    if (bg) cudaStreamSynchronize(bg);
    for (auto g : vgraphs)
        if (g) cudaGraphExecDestroy(g);
    if (apply_graph) cudaGraphExecDestroy(apply_graph);
    if (ev_jdone) cudaEventDestroy(ev_jdone);
    if (ev_applied) cudaEventDestroy(ev_applied);
    if (bg) cudaStreamDestroy(bg);
    lr_free(*this);
    for (auto e : ev_act) cudaEventDestroy(e);
    for (auto e : step_ev) cudaEventDestroy(e);
    if (ev_t0) cudaEventDestroy(ev_t0);
    dfree(params);
    dfree(wshadow);
    dfree(grads);
    for (void* p : acts) dfree(p);
    dfree(zout);
    for (void* p : dz) dfree(p);
    for (float* p : r_in) dfree(p);
    for (float* p : r_out) dfree(p);
    ng_free(*this);
    dfree(scal);
    dfree(d_step);
    dfree(d_lr);
    dfree(d_rows);
    dfree(d_ybatch);
    dfree(ce_rows);
    dfree(d_ce);
    dfree(d_flags);
    dfree(d_err);
    dfree(eval_rows);
    dfree(eval_correct);
    for (auto e : ev_bwd) cudaEventDestroy(e);
    for (auto e : ev_dw) cudaEventDestroy(e);
    for (auto e : ev_upd) cudaEventDestroy(e);
    for (auto e : ev_gate) cudaEventDestroy(e);
    if (ev_tail) cudaEventDestroy(ev_tail);
    if (ev_side) cudaEventDestroy(ev_side);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
}

void Replica::sync_shadow(cudaStream_t s) {
    if (!wshadow) return;
    for (int l = 0; l < L; ++l)
        launch_f32_to_bf16_rows(params + w_off[l], ldw[l], dims[l + 1], dims[l], wshadow + w_off[l], s);
}

void Replica::set_params(const double* flat) {
    std::vector<float> h(static_cast<size_t>(n_pad), 0.f);
    long pos = 0;
    for (int l = 0; l < L; ++l) {
        for (long r = 0; r < dims[l + 1]; ++r)
            for (long c = 0; c < dims[l]; ++c) h[w_off[l] + r * ldw[l] + c] = static_cast<float>(flat[pos++]);
        for (long r = 0; r < dims[l + 1]; ++r) h[b_off[l] + r] = static_cast<float>(flat[pos++]);
    }
    CUDA_THROW(cudaSetDevice(ctx->device));
    CUDA_THROW(cudaStreamSynchronize(stream));
    CUDA_THROW(cudaStreamSynchronize(ctx->avg));
    upload(params, h.data(), h.size() * 4);
    sync_shadow(stream);
    CUDA_THROW(cudaStreamSynchronize(stream));
}

void Replica::get_params(double* flat) const {
    std::vector<float> h(static_cast<size_t>(n_pad));
    CUDA_THROW(cudaSetDevice(ctx->device));
    CUDA_THROW(cudaStreamSynchronize(stream));
    CUDA_THROW(cudaStreamSynchronize(ctx->avg));  // a pending average
    CUDA_THROW(cudaMemcpy(h.data(), params, h.size() * 4, cudaMemcpyDeviceToHost));
    long pos = 0;
    for (int l = 0; l < L; ++l) {
        for (long r = 0; r < dims[l + 1]; ++r)
            for (long c = 0; c < dims[l]; ++c) flat[pos++] = h[w_off[l] + r * ldw[l] + c];
        for (long r = 0; r < dims[l + 1]; ++r) flat[pos++] = h[b_off[l] + r];
    }
}

// factors: per layer r_in (din x din) then r_out (dout x dout), row-major.
void Replica::get_ng_state(double* f) const {
    if (opt != OPT_NG_KRON) throw std::runtime_error("replica: not an NG-SGD replica");
    CUDA_THROW(cudaStreamSynchronize(stream));
    long pos = 0;
    for (int l = 0; l < L; ++l) {
        for (int side = 0; side < 2; ++side) {
            const long n = side == 0 ? dims[l] : dims[l + 1];
            const long ld = pad32(n);
            std::vector<float> h(static_cast<size_t>(n * ld));
            CUDA_THROW(cudaMemcpy(h.data(), side == 0 ? r_in[l] : r_out[l], h.size() * 4, cudaMemcpyDeviceToHost));
            for (long i = 0; i < n; ++i)
                for (long j = 0; j < n; ++j) f[pos++] = h[i * ld + j];
        }
    }
}

void Replica::set_ng_state(const double* f, long t) {
    if (opt != OPT_NG_KRON) throw std::runtime_error("replica: not an NG-SGD replica");
    long pos = 0;
    for (int l = 0; l < L; ++l) {
        for (int side = 0; side < 2; ++side) {
            const long n = side == 0 ? dims[l] : dims[l + 1];
            const long ld = pad32(n);
            std::vector<float> h(static_cast<size_t>(n * ld), 0.f);
            for (long i = 0; i < n; ++i)
                for (long j = 0; j < n; ++j) h[i * ld + j] = static_cast<float>(f[pos++]);
            upload(side == 0 ? r_in[l] : r_out[l], h.data(), h.size() * 4);
        }
    }
    ng_t = t;
    long tt = t;
    upload(reinterpret_cast<char*>(scal) + 8 * (16 * (L + 1) + 500), &tt, 8);
}

void Replica::bind(DeviceDataset* ds) {
    if (ds->d != dims[0])
        throw std::runtime_error("forward: input has " + std::to_string(ds->d) + " columns, model expects " +
                                 std::to_string(dims[0]));
    if (ds->classes > dims[L])
        throw std::runtime_error("dataset: " + std::to_string(ds->classes) + " classes exceed output dim " +
                                 std::to_string(dims[L]));
    bound = ds;
    ds->features(prec);  // materialise the operand-typed copy before graph capture
    const bool F = f32();
    const int sms = ctx->num_sms;
    fwd.assign(L, GemmPlan());
    dw.assign(L, GemmPlan());
    da.assign(L, GemmPlan());
    mom_in.assign(L, GemmPlan());
    mom_out.assign(L, GemmPlan());
    float* coef = reinterpret_cast<float*>(scal + 16 * (L + 1) + 480);
    static const bool no_group = [] {
        const char* v = std::getenv("PARNN_NO_DW_GROUP");
        return v && v[0] == '1';
    }();
    // bf16 dW plans use the group's tile shape (BN = 256) even when launched per layer,
    // so both launch forms compute identical tiles (tests/test_gpu.py)
    const bool group_dw = !F && (opt == OPT_SGD || opt == OPT_NG_LOWRANK) && L <= kGroupMax;
    for (int l = 0; l < L; ++l) {
        const long din = dims[l], dout = dims[l + 1];
        const void* W = F ? static_cast<const void*>(params + w_off[l]) : static_cast<const void*>(wshadow + w_off[l]);
        GemmEpi e;
        e.act = act;
        if (l + 1 < L) {
            e.mode = EPI_FWD_ACT;
            e.out = acts[l + 1];
            e.ld_out = ld_act[l + 1];
        } else {
            e.mode = EPI_FWD_LINEAR;
            e.out32 = zout;
            e.ld_out32 = ld_act[L];
        }
        e.bias = params + b_off[l];
        gemm_plan(fwd[l], prec, false, acts[l], ld_act[l], false, W, ldw[l], B, dout, din, e, sms);

        // dW = dz^T A_prev / B  (M = dout, N = din, K = B)
        GemmEpi g;
        g.alpha = 1.f / static_cast<float>(B);
        g.flag = d_flags;
        g.flag_bit = 2 * l;
        if (opt == OPT_SGD || opt == OPT_NG_LOWRANK) {
            g.mode = EPI_GRAD_SGD;
            g.out32 = params + w_off[l];
            g.ld_out32 = ldw[l];
            g.shadow = wshadow ? wshadow + w_off[l] : nullptr;
            g.ld_shadow = ldw[l];
            g.lr = d_lr;
            g.step = d_step;
        } else {
            g.mode = EPI_GRAD;
            g.out32 = grads + w_off[l];
            g.ld_out32 = ldw[l];
        }
        if (opt == OPT_NG_LOWRANK) {
            // [dW | db] = g_in g_out / B  Dhat^T [Ahat | ahat_1]  (preconditioned vectors; the
            // extra column din of the input side's xhat is its preconditioned ones column)
            LrSide& si = lrl[l].in;
            LrSide& so = lrl[l].out;
            g.gscale_a = si.st + 2 * si.R + 2;
            g.gscale_b = so.st + 2 * so.R + 2;
            g.bias_col = static_cast<int>(din);
            g.bias32 = params + b_off[l];
            gemm_plan(dw[l], prec, true, so.xhat, so.ldxh, true, si.xhat, si.ldxh, dout, din + 1, B, g, sms,
                      group_dw ? 256 : 0);
        } else if (bias_in_dw) {
            // [dW | db] = dz^T [A_prev | 1] / B: the ones column's output is the bias gradient
            g.bias_col = static_cast<int>(din);
            g.bias32 = params + b_off[l];
            gemm_plan(dw[l], prec, true, dz[l], ld_act[l + 1], true, acts[l], ld_act[l], dout, din + 1, B, g, sms,
                      group_dw ? 256 : 0);
        } else {
            gemm_plan(dw[l], prec, true, dz[l], ld_act[l + 1], true, acts[l], ld_act[l], dout, din, B, g, sms,
                      group_dw ? 256 : 0);
        }

        if (l > 0) {
            // dz_{l-1} = (dz_l W_l) * act'(A_{l-1})   (M = B, N = din, K = dout)
            GemmEpi a;
            a.mode = EPI_ACTGRAD;
            a.act = act;
            a.out = dz[l - 1];
            a.ld_out = ld_act[l];
            a.aux = acts[l];
            a.ld_aux = ld_act[l];
            gemm_plan(da[l], prec, false, dz[l], ld_act[l + 1], true, W, ldw[l], B, din, dout, a, sms);
        }
        if (opt == OPT_NG_KRON) {
            GemmEpi m;
            m.mode = EPI_EMA;
            m.coef = coef;
            m.out32 = r_in[l];
            m.ld_out32 = pad32(din);
            gemm_plan(mom_in[l], prec, true, acts[l], ld_act[l], true, acts[l], ld_act[l], din, din, B, m, sms);
            m.out32 = r_out[l];
            m.ld_out32 = pad32(dout);
            gemm_plan(mom_out[l], prec, true, dz[l], ld_act[l + 1], true, dz[l], ld_act[l + 1], dout, dout, B, m, sms);
        }
    }
    dw_group = group_dw && !no_group;
    if (dw_group) {
        std::vector<const GemmPlan*> parts;
        for (int l = L - 1; l >= 0; --l) parts.push_back(&dw[l]);  // the largest (output) layer first
        for (auto* p : parts) dw_group = dw_group && gemm_groupable(*p);
        if (dw_group) gemm_group_plan(dwg, parts, sms);
    }
    if (opt == OPT_NG_KRON) ng_build_plans(*this);
    if (opt == OPT_NG_LOWRANK) lr_build_plans(*this);
    graph = nullptr;  // an alias of vgraphs[0] (destroyed below)
    for (auto& g : vgraphs)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    vgraphs.assign(kVariants, nullptr);
    vnodes.assign(kVariants, 0);
    if (opt == OPT_NG_LOWRANK && !bg) {
        bg = make_stream(2);  // background subspace updates fill the gaps
        CUDA_THROW(cudaEventCreateWithFlags(&ev_jdone, cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&ev_applied, cudaEventDisableTiming));
    }
    if (bg) CUDA_THROW(cudaStreamSynchronize(bg));
    apply_pending = false;
    if (std::getenv("PARNN_NO_GRAPH")) use_graph = false;  // debugging: eager launches
    tl.clear();
    if (std::getenv("PARNN_TIMELINE") && tl_pool.empty()) {
        tl_pool.resize(128);
        for (auto& e : tl_pool) CUDA_THROW(cudaEventCreate(&e));
    }
    if (use_graph) {
        if (opt == OPT_NG_LOWRANK) {
            // one graph per step kind (captured here for the first two update periods,
            // others on first use); kernels_per_step = average over one period
            const int P = std::max(1, lrc.update_period);
            for (long t = 0; t < 2 * P + 3; ++t) {
                const int v = lr_variant(t);
                if (!vgraphs[v]) capture_variant(v);
            }
            if (lr_lag() >= 2) {
                if (apply_graph) cudaGraphExecDestroy(apply_graph);
                apply_graph = nullptr;
                capture_apply_graph();
            }
            long sum = 0;
            for (long t = 2 * P; t < 3 * P; ++t) sum += vnodes[lr_variant(t)];
            if (lr_lag() >= 2) sum += apply_nodes;
            kernels_per_step = sum / P;
        } else {
            capture_variant(0);  // the plain step; gated variants are captured on first use
            graph = vgraphs[0];
            kernels_per_step = vnodes[0];
        }
    }
}

void Replica::capture_variant(int v) {
    const int saved = variant;
    variant = v;
    cudaGraph_t g;
    CUDA_THROW(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_step(stream);
    } catch (...) {
        cudaStreamEndCapture(stream, &g);
        variant = saved;
        throw;
    }
    CUDA_THROW(cudaStreamEndCapture(stream, &g));
    vnodes[v] = count_kernel_nodes(g);
    CUDA_THROW(cudaGraphInstantiate(&vgraphs[v], g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    variant = saved;
}

void Replica::precapture_gates() {
    if (!use_graph || !bound) return;
    std::vector<int> base{0};
    if (opt == OPT_NG_LOWRANK) {
        base.clear();
        const int P = std::max(1, lrc.update_period);
        for (long t = 0; t < 3 * P + 3; ++t) {
            const int v = lr_variant(t);
            if (std::find(base.begin(), base.end(), v) == base.end()) base.push_back(v);
        }
    }
    for (int b : base)
        for (int g : {static_cast<int>(GATE_WAIT), static_cast<int>(GATE_REC), GATE_WAIT | GATE_REC})
            if (!vgraphs[b | g]) capture_variant(b | g);
}

// lag >= 2 low-rank updates: the step that commits a background update waits for it
void Replica::lr_before_step(cudaStream_t s) {
    if ((variant & LRV_COMMIT) && apply_pending) {
        CUDA_THROW(cudaStreamWaitEvent(s, ev_applied, 0));
        apply_pending = false;
    }
}

// ...and the step that computed J launches it on the background stream
void Replica::lr_after_step(cudaStream_t s) {
    if (lr_lag() < 2 || !(variant & LRV_J) || prof) return;
    CUDA_THROW(cudaEventRecord(ev_jdone, s));
    CUDA_THROW(cudaStreamWaitEvent(bg, ev_jdone, 0));
    if (use_graph && apply_graph) {
        CUDA_THROW(cudaGraphLaunch(apply_graph, bg));
    } else {
        for (int l = L - 1; l >= 0; --l) {
            lr_apply_update(*this, lrl[l].out, bg);
            lr_apply_update(*this, lrl[l].in, bg);
        }
    }
    CUDA_THROW(cudaEventRecord(ev_applied, bg));
    apply_pending = true;
}

void Replica::capture_apply_graph() {
    // every side's update as an independent branch, largest (out side, last layer) first
    cudaGraph_t g;
    CUDA_THROW(cudaStreamBeginCapture(bg, cudaStreamCaptureModeThreadLocal));
    try {
        CUDA_THROW(cudaEventRecord(ev_t0, bg));
        for (int pass = 0; pass < 2; ++pass)
            for (int l = L - 1; l >= 0; --l) {
                LrSide& sd = pass == 0 ? lrl[l].out : lrl[l].in;
                CUDA_THROW(cudaStreamWaitEvent(sd.stream, ev_t0, 0));
                lr_apply_update(*this, sd, sd.stream);
                CUDA_THROW(cudaEventRecord(sd.done, sd.stream));
            }
        for (int l = 0; l < L; ++l) {
            CUDA_THROW(cudaStreamWaitEvent(bg, lrl[l].in.done, 0));
            CUDA_THROW(cudaStreamWaitEvent(bg, lrl[l].out.done, 0));
        }
    } catch (...) {
        cudaStreamEndCapture(bg, &g);
        throw;
    }
    CUDA_THROW(cudaStreamEndCapture(bg, &g));
    apply_nodes = count_kernel_nodes(g);
    CUDA_THROW(cudaGraphInstantiate(&apply_graph, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
}

void Replica::tmark(const std::string& name, cudaStream_t s) {
    if (tl.size() >= tl_pool.size()) return;
    cudaEvent_t e = tl_pool[tl.size()];
    // External: becomes an event-record node of the captured graph (a plain
    // record inside a capture is only a fork/join marker)
    cudaStreamCaptureStatus cs;
    CUDA_THROW(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        CUDA_THROW(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else
        CUDA_THROW(cudaEventRecord(e, s));
    tl.emplace_back(name, e);
}

void Replica::dump_timeline() {
    if (tl.empty()) return;
    std::ostringstream os;
    os << "[parnn timeline ms]";
    for (auto& [name, e] : tl) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, tl[0].second, e) == cudaSuccess) os << " " << name << "=" << t;
    }
    fprintf(stderr, "%s\n", os.str().c_str());
}

void Replica::mark(const char* kind, int layer, double flops, cudaStream_t s) {
    if (!prof) return;
    cudaEvent_t e;
    CUDA_THROW(cudaEventCreate(&e));
    CUDA_THROW(cudaEventRecord(e, s));
    prof->events.push_back(e);
    prof->names.push_back(std::string(kind) + ":" + std::to_string(layer));
    prof->flops.push_back(flops);
}

namespace {

// One side's in-step chain on its own stream: [init updates], precondition,
// [J of the update applied at the start of the next step].
void lr_side_chain(Replica& r, LrSide& sd, cudaEvent_t wait, cudaStream_t ss) {
    if (wait) CUDA_THROW(cudaStreamWaitEvent(ss, wait, 0));
    if (r.variant & LRV_INIT)
        for (int it = 0; it < r.lrc.init_iters; ++it) {
            lr_precondition_side(r, sd, ss);
            lr_start_update(r, sd, ss);
            lr_apply_update(r, sd, ss);
            lr_commit_update(r, sd, ss);
        }
    // timing aid: PARNN_LR_SKIP=1 (in sides) / 2 (out sides) / 3 drops the precondition work
    static const int skip = std::getenv("PARNN_LR_SKIP") ? std::atoi(std::getenv("PARNN_LR_SKIP")) : 0;
    if (!(skip & (sd.in ? 1 : 2))) lr_precondition_side(r, sd, ss);
    CUDA_THROW(cudaEventRecord(sd.ready, ss));
    if (r.variant & LRV_J) {
        lr_start_update(r, sd, ss);
        // profiled lag-2 steps compute the update inline (no background graph)
        if (r.prof && r.lr_lag() >= 2) lr_apply_update(r, sd, ss);
    }
    CUDA_THROW(cudaEventRecord(sd.done, ss));
}

// The low-rank NG step. Concurrency: the pending subspace updates run from
// t0 alongside the forward pass; each layer's in-side chain starts as soon
// as the forward has produced its input, each out-side chain as soon as the
// backward has produced its dz; dW_l (+ bias) runs on the side stream once
// dA_l has read W_l and both sides of layer l are preconditioned.
void enqueue_lowrank(Replica& r, cudaStream_t s) {
    // beside a background subspace update (one long CTA per side) the GEMM grids
    // leave 2L SMs free, so no GEMM CTA queues behind an eigensolve
    struct Cap {
        explicit Cap(int c) { gemm_set_grid_cap(c); }
        ~Cap() { gemm_set_grid_cap(0); }
    } cap((r.variant & LRV_INFLIGHT) && !r.prof ? r.ctx->num_sms - 2 * r.L : 0);
    const bool F = r.f32();
    const int L = r.L;
    DeviceDataset* ds = r.bound;
    auto gf = [](const GemmPlan& p) { return 2.0 * p.M * p.N * p.K; };
    if (r.prof) {
        // profiled: serial on one stream so event regions are well defined
        r.mark("start", -1, 0, s);
        if (r.variant & (LRV_APPLY | LRV_COMMIT)) {
            for (int l = 0; l < L; ++l)
                for (LrSide* sd : {&r.lrl[l].in, &r.lrl[l].out}) {
                    if (r.variant & LRV_APPLY) lr_apply_update(r, *sd, s);
                    lr_commit_update(r, *sd, s);
                }
            r.mark("ng_lr_apply", -1, 0, s);
        }
        launch_gather(ds->features(r.prec), ds->ld, ds->y, r.d_rows, r.d_step, r.B, r.dims[0], r.acts[0],
                      r.ld_act[0], r.d_ybatch, F, s);
        r.mark("gather", 0, 0, s);
        for (int l = 0; l < L; ++l) {
            if (r.variant & GATE_WAIT) wait_ext(s, r.ev_gate[l]);
            gemm_launch(r.fwd[l], s);
            r.mark("gemm_fwd", l, gf(r.fwd[l]), s);
        }
        launch_softmax_ce(r.zout, r.ld_act[L], r.B, r.dims[L], r.d_ybatch, r.dz[L - 1], r.ld_act[L], r.ce_rows, F, s);
        r.mark("softmax_ce", L - 1, 0, s);
        for (int l = L - 1; l > 0; --l) {
            gemm_launch(r.da[l], s);
            r.mark("gemm_da", l, gf(r.da[l]), s);
        }
        double dwf = 0.0;
        for (int l = L - 1; l >= 0; --l) {
            lr_side_chain(r, r.lrl[l].in, nullptr, s);
            lr_side_chain(r, r.lrl[l].out, nullptr, s);
            r.mark("ng_lr_precondition", l, 0, s);
            dwf += gf(r.dw[l]);
            if (r.dw_group) continue;
            lr_layer_update(r, l, s);
            if (r.variant & GATE_REC) record_ext(r.ev_upd[l], s);
            r.mark("gemm_dw_sgd", l, gf(r.dw[l]), s);
        }
        if (r.dw_group) {
            gemm_group_launch(r.dwg, s);
            if (r.variant & GATE_REC)
                for (int l = 0; l < L; ++l) record_ext(r.ev_upd[l], s);
            r.mark("gemm_dw_sgd", -1, dwf, s);  // all layers, one grouped launch
        }
    } else {
        static const bool serial = std::getenv("PARNN_LR_SERIAL") != nullptr;  // debugging: one stream
        auto S = [&](cudaStream_t x) { return serial ? s : x; };
        r.tmark("t0", s);
        CUDA_THROW(cudaEventRecord(r.ev_t0, s));
        for (int l = 0; l < L; ++l)
            for (LrSide* sd : {&r.lrl[l].in, &r.lrl[l].out}) {
                CUDA_THROW(cudaStreamWaitEvent(S(sd->stream), r.ev_t0, 0));
                if (r.variant & LRV_APPLY) lr_apply_update(r, *sd, S(sd->stream));
                if (r.variant & (LRV_APPLY | LRV_COMMIT)) lr_commit_update(r, *sd, S(sd->stream));
            }
        launch_gather(ds->features(r.prec), ds->ld, ds->y, r.d_rows, r.d_step, r.B, r.dims[0], r.acts[0],
                      r.ld_act[0], r.d_ybatch, F, s);
        static const int in_late = [] {  // tuning aid: input-side chains 0 = beside the forward, 1 = from the loss on
            const char* v = std::getenv("PARNN_LR_IN_LATE");
            return v ? std::atoi(v) : 0;
        }();
        CUDA_THROW(cudaEventRecord(r.ev_act[0], s));
        // the gather's successors start ~8 us late as programmatic dependents in this
        // graph (measured; not so in the SGD step): plain launches for them
        static const int pdl_head = [] {
            const char* v = std::getenv("PARNN_LR_PDL_HEAD");
            return v ? std::atoi(v) : 0;
        }();
        gemm_set_pdl(pdl_head != 0);
        if (!in_late) lr_side_chain(r, r.lrl[0].in, r.ev_act[0], S(r.lrl[0].in.stream));
        for (int l = 0; l < L; ++l) {
            if (r.variant & GATE_WAIT) wait_ext(s, r.ev_gate[l]);  // layer l's pending average is done
            gemm_launch(r.fwd[l], s);
            gemm_set_pdl(true);
            if (l + 1 < L) {
                CUDA_THROW(cudaEventRecord(r.ev_act[l + 1], s));
                if (!in_late) lr_side_chain(r, r.lrl[l + 1].in, r.ev_act[l + 1], S(r.lrl[l + 1].in.stream));
            }
        }
        launch_softmax_ce(r.zout, r.ld_act[L], r.B, r.dims[L], r.d_ybatch, r.dz[L - 1], r.ld_act[L], r.ce_rows, F, s);
        r.tmark("fwd", s);
        CUDA_THROW(cudaEventRecord(r.ev_dw[L - 1], s));  // dz[L-1] ready
        if (in_late)
            for (int l = L - 1; l >= 0; --l) lr_side_chain(r, r.lrl[l].in, r.ev_dw[L - 1], S(r.lrl[l].in.stream));
        {
            // the step's loss is reduced beside the backward (the step counter advances at the end)
            cudaStream_t os = S(r.lrl[L - 1].out.stream);
            CUDA_THROW(cudaStreamWaitEvent(os, r.ev_dw[L - 1], 0));
            launch_ce_reduce(r.ce_rows, r.B, r.d_ce, r.d_step, 0, os);
        }
        lr_side_chain(r, r.lrl[L - 1].out, r.ev_dw[L - 1], S(r.lrl[L - 1].out.stream));
        for (int l = L - 1; l >= 0; --l) {
            if (l > 0) gemm_launch(r.da[l], s);
            CUDA_THROW(cudaEventRecord(r.ev_bwd[l], s));  // W_l read; dz[l-1] ready
            if (l > 0) lr_side_chain(r, r.lrl[l - 1].out, r.ev_bwd[l], S(r.lrl[l - 1].out.stream));
        }
        if (r.dw_group) {
            // [dW_l | db_l] of every layer in one grouped persistent launch once the dz
            // chain and every side's preconditioning are done: the epilogues (the fp32
            // weight read-modify-write) of one layer's tiles overlap the mainloops of others
            for (int l = 0; l < L; ++l) {
                CUDA_THROW(cudaStreamWaitEvent(s, r.lrl[l].in.ready, 0));
                CUDA_THROW(cudaStreamWaitEvent(s, r.lrl[l].out.ready, 0));
            }
            gemm_group_launch(r.dwg, s);
            r.tmark("dw", s);
            if (r.variant & GATE_REC)
                for (int l = 0; l < L; ++l) record_ext(r.ev_upd[l], s);
        }
        for (int l = L - 1; l >= 0 && !r.dw_group; --l) {
            // [dW_l | db_l] on the layer's input-side stream: the layers' weight updates are
            // independent and overlap each other and the remaining chains (a single side
            // stream made them the step's critical path). They start after the whole dz
            // chain: a persistent dW grid launched beside it held the SMs the next dA
            // needed (the output layer's 75 us dW delayed dA_1 by ~60 us).
            cudaStream_t ws = S(r.lrl[l].in.stream);
            CUDA_THROW(cudaStreamWaitEvent(ws, r.ev_bwd[0], 0));
            CUDA_THROW(cudaStreamWaitEvent(ws, r.lrl[l].out.ready, 0));
            lr_layer_update(r, l, ws);
            if (r.variant & GATE_REC) record_ext(r.ev_upd[l], ws);  // layer l final: its average may start
            r.tmark("dw" + std::to_string(l), ws);
            CUDA_THROW(cudaEventRecord(r.lrl[l].in.done, ws));
        }
        for (int l = 0; l < L; ++l) {
            CUDA_THROW(cudaStreamWaitEvent(s, r.lrl[l].in.done, 0));
            CUDA_THROW(cudaStreamWaitEvent(s, r.lrl[l].out.done, 0));
        }
    }
    if (r.prof) {
        flags_latch_kernel<<<1, 1, 0, s>>>(r.d_flags, r.d_step);
        launch_ce_reduce(r.ce_rows, r.B, r.d_ce, r.d_step, 1, s);
        r.mark("ce_reduce", 0, 0, s);
    } else {
        flags_latch_advance_kernel<<<1, 1, 0, s>>>(r.d_flags, r.d_step);
    }
    CUDA_THROW(cudaGetLastError());
    r.tmark("end", s);
}

}  // namespace

void Replica::enqueue_step(cudaStream_t s) {
    if (opt == OPT_NG_LOWRANK) {
        enqueue_lowrank(*this, s);
        return;
    }
    const bool F = f32();
    DeviceDataset* ds = bound;
    auto gf = [](const GemmPlan& p) { return 2.0 * p.M * p.N * p.K; };
    mark("start", -1, 0, s);
    if (!prof) tmark("t0", s);
    launch_gather(ds->features(prec), ds->ld, ds->y, d_rows, d_step, B, dims[0], acts[0], ld_act[0], d_ybatch, F, s,
                  ones_col0());
    mark("gather", 0, 0, s);
    for (int l = 0; l < L; ++l) {
        if (variant & GATE_WAIT) wait_ext(s, ev_gate[l]);  // layer l's pending average is done
        gemm_launch(fwd[l], s);
        mark("gemm_fwd", l, gf(fwd[l]), s);
    }
    launch_softmax_ce(zout, ld_act[L], B, dims[L], d_ybatch, dz[L - 1], ld_act[L], ce_rows, F, s);
    mark("softmax_ce", L - 1, 0, s);
    const bool ng = opt == OPT_NG_KRON;
    float* coef = reinterpret_cast<float*>(scal + 16 * (L + 1) + 480);
    long* tdev = reinterpret_cast<long*>(scal + 16 * (L + 1) + 500);
    if (!prof) {
        // Concurrent backward: dA_l stays on the main stream (it carries the
        // dz chain), dW_l goes to the side stream as soon as dA_l has read W_l
        // (SGD) / dz_l exists (NG); layer l's NG chain starts right after dW_l,
        // so the output layer's long Cholesky/TRSM chain overlaps the rest of
        // the backward pass.
        tmark("fwd", s);
        if (ng) ng_coeff_kernel<<<1, 1, 0, s>>>(tdev, ng_decay, 1.0 / static_cast<double>(B), coef);
        for (int l = L - 1; l >= 0; --l) {
            if (l > 0) gemm_launch(da[l], s);
            CUDA_THROW(cudaEventRecord(ev_bwd[l], s));
            CUDA_THROW(cudaStreamWaitEvent(side, ev_bwd[l], 0));
            // the bias gradient is off the dz chain: side stream, before dW_l (bf16 SGD:
            // in the dW GEMM's ones column instead)
            if (!bias_in_dw)
                launch_bias_grad(dz[l], ld_act[l + 1], B, dims[l + 1], F, ng ? nullptr : params + b_off[l],
                                 ng ? grads + b_off[l] : nullptr, d_lr, d_step, d_flags, 2 * l + 1, side);
            if (dw_group) continue;  // every layer's dW below, one grouped launch
            gemm_launch(dw[l], side);
            if (!ng && (variant & GATE_REC)) record_ext(ev_upd[l], side);  // layer l final for this step
            tmark("dw" + std::to_string(l), side);
            if (ng) {
                CUDA_THROW(cudaEventRecord(ev_dw[l], side));
                cudaStream_t ls = ngl[l].stream;
                CUDA_THROW(cudaStreamWaitEvent(ls, ev_dw[l], 0));
                gemm_launch(mom_in[l], ls);
                gemm_launch(mom_out[l], ls);
                ng_precondition_layer(*this, l, ls);
                ng_apply_update(*this, l, ls);
                if (variant & GATE_REC) record_ext(ev_upd[l], ls);
                tmark("done" + std::to_string(l), ls);
                CUDA_THROW(cudaEventRecord(ngl[l].done, ls));
            }
        }
        // grouped dW + SGD of every layer right behind the dz chain (PDL from the last dA):
        // one persistent grid, the weight read-modify-write epilogues of one layer's tiles
        // overlapping the mainloops of the next
        if (dw_group) gemm_group_launch(dwg, s);
        CUDA_THROW(cudaEventRecord(ev_side, side));
        CUDA_THROW(cudaStreamWaitEvent(s, ev_side, 0));
        if (dw_group && (variant & GATE_REC))
            for (int l = 0; l < L; ++l) record_ext(ev_upd[l], s);
        if (ng)
            for (int l = 0; l < L; ++l) CUDA_THROW(cudaStreamWaitEvent(s, ngl[l].done, 0));
        flags_latch_kernel<<<1, 1, 0, s>>>(d_flags, d_step);
        launch_ce_reduce(ce_rows, B, d_ce, d_step, 1, s);
        tmark("end", s);
        return;
    }
    for (int l = L - 1; l >= 0; --l) {
        if (!bias_in_dw) {
            launch_bias_grad(dz[l], ld_act[l + 1], B, dims[l + 1], F, ng ? nullptr : params + b_off[l],
                             ng ? grads + b_off[l] : nullptr, d_lr, d_step, d_flags, 2 * l + 1, s);
            mark("bias_grad", l, 0, s);
        }
        if (l > 0) {
            gemm_launch(da[l], s);  // reads W_l before its update below
            mark("gemm_da", l, gf(da[l]), s);
        }
        if (dw_group) continue;
        gemm_launch(dw[l], s);
        if (!ng && (variant & GATE_REC)) record_ext(ev_upd[l], s);
        mark(ng ? "gemm_dw" : "gemm_dw_sgd", l, gf(dw[l]), s);
    }
    if (dw_group) {
        double dwf = 0.0;
        for (int l = 0; l < L; ++l) dwf += gf(dw[l]);
        gemm_group_launch(dwg, s);
        if (variant & GATE_REC)
            for (int l = 0; l < L; ++l) record_ext(ev_upd[l], s);
        mark("gemm_dw_sgd", -1, dwf, s);  // all layers, one grouped launch
    }
    if (ng) {
        ng_coeff_kernel<<<1, 1, 0, s>>>(tdev, ng_decay, 1.0 / static_cast<double>(B), coef);
        if (prof) {  // profiled: serial on one stream so event regions are well defined
            for (int l = 0; l < L; ++l) {
                gemm_launch(mom_in[l], s);
                gemm_launch(mom_out[l], s);
                mark("gemm_ng_moments", l, gf(mom_in[l]) + gf(mom_out[l]), s);
            }
            for (int l = 0; l < L; ++l) {
                ng_precondition_layer(*this, l, s);
                ng_apply_update(*this, l, s);
                if (variant & GATE_REC) record_ext(ev_upd[l], s);
            }
        } else {
            // the layers' NG chains are independent: fork one stream per layer, join
            CUDA_THROW(cudaEventRecord(ng_fork, s));
            for (int l = L - 1; l >= 0; --l) {  // largest (output) layer first
                cudaStream_t ls = ngl[l].stream;
                CUDA_THROW(cudaStreamWaitEvent(ls, ng_fork, 0));
                gemm_launch(mom_in[l], ls);
                gemm_launch(mom_out[l], ls);
                ng_precondition_layer(*this, l, ls);
                ng_apply_update(*this, l, ls);
                if (variant & GATE_REC) record_ext(ev_upd[l], ls);
                CUDA_THROW(cudaEventRecord(ngl[l].done, ls));
            }
            for (int l = 0; l < L; ++l) CUDA_THROW(cudaStreamWaitEvent(s, ngl[l].done, 0));
        }
    }
    flags_latch_kernel<<<1, 1, 0, s>>>(d_flags, d_step);
    launch_ce_reduce(ce_rows, B, d_ce, d_step, 1, s);
    mark("ce_reduce", 0, 0, s);
}

void Replica::profile_steps(long steps, std::vector<std::string>& names, std::vector<double>& ms,
                            std::vector<double>& flops) {
    if (!bound) throw std::runtime_error("replica: no dataset bound");
    names.clear();
    ms.clear();
    flops.clear();
    for (long it = 0; it < steps; ++it) {
        Profile p;
        variant = gate_pending ? GATE_WAIT : 0;
        gate_pending = false;
        last_recorded = false;
        if (opt == OPT_NG_LOWRANK) {
            variant |= lr_variant(lr_t++);
            lr_before_step(stream);
        }
        prof = &p;
        try {
            enqueue_step(stream);
        } catch (...) {
            prof = nullptr;
            throw;
        }
        prof = nullptr;
        if (!step_ev.empty()) CUDA_THROW(cudaEventRecord(step_ev[epoch_steps % kStepRing], stream));
        ++epoch_steps;
        CUDA_THROW(cudaStreamSynchronize(stream));
        // accumulate by region name: step kinds (low-rank init / update / plain) differ in regions
        for (size_t i = 1; i < p.events.size(); ++i) {
            float t = 0.f;
            CUDA_THROW(cudaEventElapsedTime(&t, p.events[i - 1], p.events[i]));
            size_t k = 0;
            while (k < names.size() && names[k] != p.names[i]) ++k;
            if (k == names.size()) {
                names.push_back(p.names[i]);
                ms.push_back(0.0);
                flops.push_back(p.flops[i]);
            }
            ms[k] += t / static_cast<double>(steps);
        }
        for (auto e : p.events) cudaEventDestroy(e);
    }
}

double Replica::time_steps(long steps) {
    cudaEvent_t a, b;
    CUDA_THROW(cudaEventCreate(&a));
    CUDA_THROW(cudaEventCreate(&b));
    CUDA_THROW(cudaEventRecord(a, stream));
    for (long i = 0; i < steps; ++i) run_step(stream);
    CUDA_THROW(cudaEventRecord(b, stream));
    CUDA_THROW(cudaEventSynchronize(b));
    float t = 0.f;
    CUDA_THROW(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return t;
}

void Replica::upload_epoch(const uint32_t* rows, const float* lrs, long steps) {
    if (steps > max_steps) throw std::runtime_error("replica: epoch has more steps than max_steps");
    cudaStream_t s = stream;
    CUDA_THROW(cudaMemcpyAsync(d_rows, rows, steps * B * 4, cudaMemcpyHostToDevice, s));
    CUDA_THROW(cudaMemcpyAsync(d_lr, lrs, steps * 4, cudaMemcpyHostToDevice, s));
    CUDA_THROW(cudaMemsetAsync(d_step, 0, 4, s));
    epoch_steps = 0;
    epoch_len = steps;
}

double Replica::step_ce(long j) {
    if (j < 0 || j >= epoch_steps) throw std::runtime_error("replica: step " + std::to_string(j) + " not launched");
    if (epoch_steps - j > kStepRing)
        CUDA_THROW(cudaStreamSynchronize(stream));  // its event slot was reused
    else
        CUDA_THROW(cudaEventSynchronize(step_ev[j % kStepRing]));
    double v = 0.0;
    CUDA_THROW(cudaMemcpy(&v, d_ce + j, sizeof(double), cudaMemcpyDeviceToHost));
    return v;
}

void Replica::run_step(cudaStream_t s, bool window_end) {
    if (!bound) throw std::runtime_error("replica: no dataset bound");
    if (epoch_steps >= epoch_len)
        throw std::runtime_error("replica: step " + std::to_string(epoch_steps) + " beyond the " +
                                 std::to_string(epoch_len) + " uploaded for this epoch");
    if (bound->written) CUDA_THROW(cudaStreamWaitEvent(s, bound->written, 0));  // inputs written by the host
    if (step_ev.empty()) {
        step_ev.resize(kStepRing);
        for (auto& e : step_ev) CUDA_THROW(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    struct Rec {
        Replica* r;
        cudaStream_t s;
        ~Rec() { cudaEventRecord(r->step_ev[r->epoch_steps++ % kStepRing], s); }
    } rec{this, s};
    const int gating = (gate_pending ? GATE_WAIT : 0) | (window_end ? GATE_REC : 0);
    gate_pending = false;
    last_recorded = window_end;
    if (opt == OPT_NG_LOWRANK) {
        variant = lr_variant(lr_t);
        static const char* force = std::getenv("PARNN_LR_FORCE_VARIANT");  // timing aid (LRV_* bits)
        if (force && lr_t > 0) variant = std::atoi(force);
        variant |= gating;
        lr_before_step(s);
        if (use_graph) {
            if (!vgraphs[variant]) capture_variant(variant);
            CUDA_THROW(cudaGraphLaunch(vgraphs[variant], s));
        } else {
            enqueue_step(s);
        }
        lr_after_step(s);
        ++lr_t;
        return;
    }
    variant = gating;
    if (use_graph) {
        if (!vgraphs[variant]) capture_variant(variant);
        CUDA_THROW(cudaGraphLaunch(vgraphs[variant], s));
    } else {
        enqueue_step(s);
    }
}

void Replica::check_errors() {
    if (!tl.empty()) {
        CUDA_THROW(cudaStreamSynchronize(stream));
        dump_timeline();
    }
    DevErr e;
    unsigned f[4];
    CUDA_THROW(cudaStreamSynchronize(stream));
    CUDA_THROW(cudaMemcpy(&e, d_err, sizeof(e), cudaMemcpyDeviceToHost));
    CUDA_THROW(cudaMemcpy(f, d_flags, sizeof(f), cudaMemcpyDeviceToHost));
    // Reference order: ng_precondition (Cholesky) throws before sgd_step's checks.
    if (e.chol_failed) {
        std::ostringstream os;
        os << "cholesky_solve: non-positive-definite pivot ";
        // the reference (x86, glibc) prints its NaN pivots as -nan (the default NaN is negative)
        if (std::isnan(e.chol_value)) os << "-nan";
        else os << e.chol_value;
        os << " at index " << e.chol_index;
        throw std::runtime_error(os.str());
    }
    const unsigned bits = f[1] | f[0];
    if (bits) {
        for (int l = 0; l < L; ++l) {
            if (bits & (1u << (2 * l))) throw std::runtime_error("sgd_step: non-finite weight gradient in layer " + std::to_string(l));
            if (bits & (1u << (2 * l + 1))) throw std::runtime_error("sgd_step: non-finite bias gradient in layer " + std::to_string(l));
        }
    }
}

double Replica::accuracy(DeviceDataset* ds) {
    if (ds->n == 0) throw std::runtime_error("accuracy: empty feature matrix");
    if (ds->d != dims[0])
        throw std::runtime_error("forward: input has " + std::to_string(ds->d) + " columns, model expects " +
                                 std::to_string(dims[0]));
    if (!bound) throw std::runtime_error("replica: bind a training dataset first");
    cudaStream_t s = stream;
    const bool F = f32();
    if (!eval_correct) eval_correct = dalloc<unsigned long long>(1);
    if (eval_rows_n < ds->n) {  // identity row ids, grown on demand and kept
        CUDA_THROW(cudaStreamSynchronize(s));
        dfree(eval_rows);
        eval_rows = dalloc<uint32_t>(ds->n);
        std::vector<uint32_t> h(ds->n);
        for (long i = 0; i < ds->n; ++i) h[i] = static_cast<uint32_t>(i);
        upload(eval_rows, h.data(), ds->n * 4);
        eval_rows_n = ds->n;
    }
    uint32_t* rows = eval_rows;
    unsigned long long* correct = eval_correct;
    CUDA_THROW(cudaMemsetAsync(correct, 0, sizeof(unsigned long long), s));
    for (int l = 0; l < L; ++l) wait_ext(s, ev_gate[l]);  // a pending average
    for (long c0 = 0; c0 < ds->n; c0 += B) {
        const long cb = std::min(B, ds->n - c0);
        launch_gather(ds->features(prec), ds->ld, ds->y, rows + c0, nullptr, cb, dims[0], acts[0], ld_act[0], d_ybatch,
                      F, s, ones_col0());
        for (int l = 0; l < L; ++l) gemm_launch(fwd[l], s);
        launch_argmax_correct(zout, ld_act[L], cb, dims[L], d_ybatch, correct, s);
    }
    unsigned long long hc = 0;
    CUDA_THROW(cudaMemcpyAsync(&hc, correct, 8, cudaMemcpyDeviceToHost, s));
    CUDA_THROW(cudaStreamSynchronize(s));
    return static_cast<double>(hc) / static_cast<double>(ds->n);
}

// Forward for `b` given dataset rows (test hook): returns the last layer's Z.
void Replica::forward_only(DeviceDataset* ds, const uint32_t* rows_h, long b, float* zh) {
    if (b > B) throw std::runtime_error("forward: batch larger than the replica's minibatch");
    cudaStream_t s = stream;
    uint32_t* rows = dalloc<uint32_t>(b);
    CUDA_THROW(cudaMemcpyAsync(rows, rows_h, b * 4, cudaMemcpyHostToDevice, s));
    for (int l = 0; l < L; ++l) wait_ext(s, ev_gate[l]);
    launch_gather(ds->features(prec), ds->ld, ds->y, rows, nullptr, b, dims[0], acts[0], ld_act[0], d_ybatch, f32(), s,
                  ones_col0());
    for (int l = 0; l < L; ++l) gemm_launch(fwd[l], s);
    std::vector<float> h(static_cast<size_t>(b * ld_act[L]));
    CUDA_THROW(cudaMemcpyAsync(h.data(), zout, h.size() * 4, cudaMemcpyDeviceToHost, s));
    CUDA_THROW(cudaStreamSynchronize(s));
    for (long i = 0; i < b; ++i)
        for (long j = 0; j < dims[L]; ++j) zh[i * dims[L] + j] = h[i * ld_act[L] + j];
    dfree(rows);
}

}  // namespace pnb
