"""Python mirror of the reference trainer API (namespace ``parnn``) over the
C ABI of libparnn_b200.so. Names, argument meaning and error behaviour follow
the reference headers:

* ``ParallelPlan``, ``TrainOptions``, ``EpochMetrics``, ``TrainResult``,
  ``train_parallel``, ``serial_train``, ``allreduce_average``,
  ``partition_data``                                      (parallel.hpp:22-81)
* ``MlpModel``, ``init_random``, ``flatten``/``unflatten``, ``accuracy``,
  ``save_model``/``load_model``, ``param_count``          (network.hpp:27-95)
* ``exponential_lr``, ``newbob_next``, ``scale_lr_for_workers``,
  ``make_schedule``                                       (optimizer.hpp:57-96)
* ``Dataset``, ``generate_synthetic``/``split_cv``/standardize,
  ``shuffled_indices``, ``minibatches``                   (data.hpp:17-69)
* ``greedy_pretrain``, ``PretrainOptions``, ``Rbm``       (pretrain.hpp:14-76)

Errors raise ``ParnnError`` carrying the reference's message text.
All arithmetic runs in the CUDA library; this module only moves host buffers.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import ParnnError, TrainConfig, check, f64, i32, lib, ptr, u64

__all__ = [
    "ParnnError", "Activation", "OptimizerKind", "LrVariant", "Precision", "Dataset", "MlpModel",
    "ParallelPlan", "TrainOptions", "EpochMetrics", "TrainResult", "PretrainOptions", "Context",
    "DeviceDataset", "Replica", "Comm", "Rbm", "rng_u64", "rng_uniform", "rng_gaussian", "shuffled_indices",
    "partition_rows", "partition_data", "minibatch_rows", "make_data", "param_count", "init_random",
    "flatten", "unflatten", "exponential_lr", "newbob_sequence", "scale_lr_for_workers", "save_model",
    "load_model", "allreduce_average", "train_parallel", "serial_train", "greedy_pretrain",
]


class Activation(enum.IntEnum):
    sigmoid = 0
    tanh = 1


class OptimizerKind(enum.IntEnum):
    sgd = 0
    ngsgd = 1          # the reference's kron-full NG-SGD (optimizer.cpp:44-157)
    ngsgd_lowrank = 2  # online low-rank NG-SGD (north star; not in the reference)


class LrVariant(enum.IntEnum):
    newbob = 0
    exponential = 1


class Precision(enum.IntEnum):
    bf16 = 0
    tf32 = 1
    fp32 = 2  # 3xTF32 split on tcgen05: fp32-accurate (parity mode)


# ------------------------------------------------------------ value types
@dataclass
class Dataset:
    features: np.ndarray  # N x D float64
    labels: np.ndarray    # N int32
    num_classes: int = 0

    def size(self) -> int:
        return int(self.features.shape[0])

    def dim(self) -> int:
        return int(self.features.shape[1])


@dataclass
class MlpModel:
    layer_dims: list
    activation: Activation = Activation.sigmoid
    params: np.ndarray = None  # canonical flatten order (network.hpp:59-66)

    def num_layers(self) -> int:
        return len(self.layer_dims) - 1


@dataclass
class ParallelPlan:
    workers: int = 1
    avg_frequency: int = 10
    minibatch: int = 128
    base_seed: int = 0


@dataclass
class TrainOptions:
    optimizer: OptimizerKind = OptimizerKind.ngsgd
    lr_schedule: LrVariant = LrVariant.exponential
    lr_init: float = 0.32
    epochs: int = 15
    ng_decay: float = 0.95
    ng_smoothing: float = 4.0
    precision: Precision = Precision.bf16  # B200 knob; bf16 operands + fp32 accumulation
    # low-rank NG-SGD knobs (optimizer ngsgd_lowrank; alpha = ng_smoothing)
    ng_rank_in: int = 20
    ng_rank_out: int = 80
    ng_update_period: int = 4
    ng_history: float = 2000.0
    ng_update_lag: int = 4


@dataclass
class EpochMetrics:
    epoch: int
    lr: float
    train_ce: float
    cv_accuracy: float
    wall_seconds: float
    workers: int
    avg_events: int


@dataclass
class TrainResult:
    model: MlpModel
    metrics: list = field(default_factory=list)
    total_wall_seconds: float = 0.0


@dataclass
class PretrainOptions:
    epochs: int = 10
    lr_gaussian: float = 0.001
    lr_bernoulli: float = 0.1
    batch_size: int = 128


# ------------------------------------------------------ host primitives
def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    check(lib().parnn_rng_u64(seed, n, ptr(out)))
    return out


def rng_uniform(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    check(lib().parnn_rng_uniform(seed, n, ptr(out)))
    return out


def rng_gaussian(seed: int, n: int, mean: float = 0.0, stddev: float = 1.0) -> np.ndarray:
    out = np.zeros(n)
    check(lib().parnn_rng_gaussian(seed, n, mean, stddev, ptr(out)))
    return out


def shuffled_indices(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    check(lib().parnn_shuffled_indices(n, seed, ptr(out)))
    return out


def partition_rows(n: int, m: int, seed: int) -> np.ndarray:
    """Row ids of each of the m shards (partition_data, parallel.cpp:61-77)."""
    if m == 0:
        check(lib().parnn_partition_rows(n, 0, seed, None))
    s = n // m if m <= n else 0
    out = np.zeros(max(m * s, 1), np.uint64)
    check(lib().parnn_partition_rows(n, m, seed, ptr(out)))
    return out[:m * s].reshape(m, s)


def partition_data(ds: Dataset, m: int, seed: int) -> list:
    rows = partition_rows(ds.size(), m, seed).astype(np.int64)
    return [Dataset(ds.features[r], ds.labels[r], ds.num_classes) for r in rows]


def minibatch_rows(n: int, batch: int, epoch_seed: int) -> np.ndarray:
    cnt = n // batch if 0 < batch <= n else 0
    out = np.zeros(max(cnt * batch, 1), np.uint64)
    check(lib().parnn_minibatch_rows(n, batch, epoch_seed, ptr(out)))
    return out[:cnt * batch].reshape(cnt, batch)


def make_data(classes: int, dim: int, per_class: int, separation: float, seed: int, cv_fraction: float = 0.10,
              split_seed: int = 0, standardize: bool = True):
    """generate_synthetic + split_cv + train-split standardization (data.cpp:124-242)."""
    n = classes * per_class
    tx = np.zeros((n, dim)); ty = np.zeros(n, np.int32)
    cx = np.zeros((n, dim)); cy = np.zeros(n, np.int32)
    ntr, ncv = C.c_uint64(), C.c_uint64()
    check(lib().parnn_make_data(classes, dim, per_class, separation, seed, cv_fraction, split_seed,
                                int(standardize), ptr(tx), ptr(ty), C.byref(ntr), ptr(cx), ptr(cy), C.byref(ncv)))
    a, b = ntr.value, ncv.value
    return Dataset(tx[:a].copy(), ty[:a].copy(), classes), Dataset(cx[:b].copy(), cy[:b].copy(), classes)


def load_csv(path: str) -> Dataset:
    """load_csv (data.cpp:66-107) on the host threads; errors carry the reference's messages."""
    n, d, k = C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(lib().parnn_load_csv(path.encode(), None, None, 0, 0, C.byref(n), C.byref(d), C.byref(k)))
    x = np.zeros((n.value, d.value))
    y = np.zeros(n.value, np.int32)
    check(lib().parnn_load_csv(path.encode(), ptr(x), ptr(y), n.value, d.value, C.byref(n), C.byref(d), C.byref(k)))
    return Dataset(x, y, k.value)


def save_csv(path: str, ds: Dataset) -> None:
    """save_csv (data.cpp:109-122)."""
    x, y = f64(ds.features), i32(ds.labels)
    check(lib().parnn_save_csv(path.encode(), ptr(x), ptr(y), x.shape[0], x.shape[1] if x.ndim == 2 else 0))


def param_count(dims) -> int:
    d = u64(dims)
    return int(lib().parnn_param_count(ptr(d), len(d)))


def init_random(dims, activation: Activation = Activation.sigmoid, seed: int = 0) -> MlpModel:
    d = u64(dims)
    p = np.zeros(max(param_count(dims), 1))
    check(lib().parnn_init_random(ptr(d), len(d), seed, ptr(p)))
    return MlpModel(list(map(int, dims)), Activation(activation), p[:param_count(dims)])


def flatten(m: MlpModel) -> np.ndarray:
    return m.params.copy()


def unflatten(p: np.ndarray, template: MlpModel) -> MlpModel:
    if p.size != param_count(template.layer_dims):
        raise ParnnError(f"unflatten: vector length {p.size} does not match model size "
                         f"{param_count(template.layer_dims)}")
    return MlpModel(list(template.layer_dims), template.activation, f64(p).copy())


def exponential_lr(lr_init: float, planned_epochs: int, progress: float) -> float:
    out = C.c_double()
    check(lib().parnn_exponential_lr(lr_init, planned_epochs, progress, C.byref(out)))
    return out.value


def newbob_sequence(lr_init: float, accs) -> tuple[np.ndarray, np.ndarray]:
    a = f64(accs)
    lr = np.zeros(max(len(a) - 1, 1)); st = np.zeros(max(len(a) - 1, 1), np.int32)
    check(lib().parnn_newbob_sequence(lr_init, ptr(a), len(a), ptr(lr), ptr(st)))
    return lr[:len(a) - 1], st[:len(a) - 1].astype(bool)


def lowrank_basis(dim: int, rank: int, seed: int) -> np.ndarray:
    """Initial orthonormal basis of the low-rank NG state (host, fp64)."""
    out = np.zeros((rank, dim))
    check(lib().parnn_lowrank_basis(dim, rank, seed, ptr(out)))
    return out


def lowrank_seed(layer: int, side: int) -> int:
    return int(lib().parnn_lowrank_seed(layer, side))


def scale_lr_for_workers(lr_init: float, workers: int) -> float:
    out = C.c_double()
    check(lib().parnn_scale_lr_for_workers(lr_init, workers, C.byref(out)))
    return out.value


def save_model(path: str, m: MlpModel) -> None:
    d = u64(m.layer_dims)
    check(lib().parnn_save_model(path.encode(), ptr(d), len(d), int(m.activation), ptr(f64(m.params))))


def load_model(path: str, max_dims: int = 64, max_params: int = 1 << 27) -> MlpModel:
    d = np.zeros(max_dims, np.uint64)
    nd = C.c_int(max_dims); act = C.c_int()
    with open(path, "rb") as f:
        head = f.read(20)
    # size the params buffer from the header when it parses; errors come from the library
    p = np.zeros(max_params if len(head) < 20 else max(1, min(max_params, 1 << 27)))
    check(lib().parnn_load_model(path.encode(), ptr(d), C.byref(nd), C.byref(act), ptr(p), p.size))
    dims = [int(v) for v in d[:nd.value]]
    return MlpModel(dims, Activation(act.value), p[:param_count(dims)].copy())


def allreduce_average(contributions, m: int) -> np.ndarray:
    """Host fixed-tree mean (parallel.cpp:40-59)."""
    if m == 0:
        raise ParnnError("allreduce_average: m must be >= 1")
    if len(contributions) != m:
        raise ParnnError(f"allreduce_average: got {len(contributions)} contributions for m = {m}")
    n = len(contributions[0])
    for r in range(1, m):
        if len(contributions[r]) != n:
            raise ParnnError(f"allreduce_average: rank {r} vector length {len(contributions[r])} differs from "
                             f"rank 0 length {n}")
    c = f64(np.stack([f64(v) for v in contributions]))
    out = np.zeros(n)
    check(lib().parnn_allreduce_average_host(ptr(c), m, n, ptr(out)))
    return out


# ------------------------------------------------------ device objects
class Context:
    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().parnn_ctx_create(device, C.byref(h)))
        self.h = h

    def sync(self):
        check(lib().parnn_ctx_sync(self.h))

    def close(self):
        if self.h:
            lib().parnn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceDataset:
    def __init__(self, ctx: Context, ds: Dataset | None = None, handle=None):
        if handle is None:
            h = C.c_void_p()
            x, y = f64(ds.features), i32(ds.labels)
            classes = ds.num_classes or (int(y.max()) + 1 if y.size else 0)
            check(lib().parnn_dataset_create(ctx.h, ptr(x), ptr(y), x.shape[0], x.shape[1], classes, C.byref(h)))
        else:
            h = handle
        self.h, self.ctx = h, ctx
        n, d, k = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().parnn_dataset_info(self.h, C.byref(n), C.byref(d), C.byref(k)))
        self.n, self.d, self.num_classes = n.value, d.value, k.value

    @staticmethod
    def generate(ctx: Context, classes: int, dim: int, per_class: int, separation: float, seed: int,
                 cv_fraction: float = 0.10, split_seed: int = 0, standardize: bool = True):
        """generate_synthetic + split_cv + standardize on the device (data.cpp:124-242):
        returns (train, cv) device datasets."""
        a, b = C.c_void_p(), C.c_void_p()
        check(lib().parnn_dataset_generate(ctx.h, classes, dim, per_class, separation, seed, cv_fraction, split_seed,
                                           int(standardize), C.byref(a), C.byref(b)))
        return DeviceDataset(ctx, handle=a), DeviceDataset(ctx, handle=b)

    @staticmethod
    def load_csv(ctx: Context, path: str):
        h = C.c_void_p()
        check(lib().parnn_dataset_load_csv(ctx.h, path.encode(), C.byref(h)))
        return DeviceDataset(ctx, handle=h)

    def download(self) -> Dataset:
        x = np.zeros((self.n, self.d), np.float32)
        y = np.zeros(self.n, np.int32)
        check(lib().parnn_dataset_download(self.h, ptr(x), ptr(y)))
        return Dataset(x, y, self.num_classes)

    def write_rows(self, x, y, row0: int = 0):
        """Host fp32 rows -> device (the per-step H2D of the end-to-end path)."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        check(lib().parnn_dataset_write_f32(self.h, ptr(x), ptr(y), row0, x.shape[0]))

    def close(self):
        if self.h:
            lib().parnn_dataset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Replica:
    """One worker (WorkerState, parallel.cpp:81-91) resident on the GPU."""

    def __init__(self, ctx: Context, dims, activation=Activation.sigmoid, precision=Precision.bf16,
                 optimizer=OptimizerKind.sgd, minibatch=128, max_steps=1, ng_decay=0.95, ng_smoothing=4.0):
        h = C.c_void_p()
        d = u64(dims)
        check(lib().parnn_replica_create(ctx.h, ptr(d), len(d), int(activation), int(precision), int(optimizer),
                                         minibatch, max_steps, ng_decay, ng_smoothing, C.byref(h)))
        self.h, self.ctx, self.dims, self.B = h, ctx, list(map(int, dims)), minibatch
        self.P = param_count(dims)

    def set_params(self, p):
        p = f64(p)
        check(lib().parnn_replica_set_params(self.h, ptr(p), p.size))

    def get_params(self) -> np.ndarray:
        out = np.zeros(self.P)
        check(lib().parnn_replica_get_params(self.h, ptr(out), self.P))
        return out

    def factor_count(self) -> int:
        d = self.dims
        return sum(d[l] ** 2 + d[l + 1] ** 2 for l in range(len(d) - 1))

    def get_ng_state(self):
        out = np.zeros(self.factor_count())
        check(lib().parnn_replica_get_ng_state(self.h, ptr(out), out.size))
        res, pos, d = [], 0, self.dims
        for l in range(len(d) - 1):
            a, b = d[l], d[l + 1]
            res.append((out[pos:pos + a * a].reshape(a, a), out[pos + a * a:pos + a * a + b * b].reshape(b, b)))
            pos += a * a + b * b
        return res

    def set_ng_state(self, factors, update_count: int):
        flat = f64(np.concatenate([np.concatenate([ri.ravel(), ro.ravel()]) for ri, ro in factors]))
        check(lib().parnn_replica_set_ng_state(self.h, ptr(flat), flat.size, update_count))

    def set_lowrank(self, rank_in: int = 20, rank_out: int = 80, update_period: int = 4, init_iters: int = 3,
                    num_samples_history: float = 2000.0, update_lag: int = 4):
        check(lib().parnn_replica_set_lowrank(self.h, rank_in, rank_out, update_period, init_iters,
                                              num_samples_history, update_lag))

    def lowrank_state(self, layer: int, side: int):
        """(W = E^1/2 R, d, rho) of one side (0 = in [A_prev | 1], 1 = out dz)."""
        rank, dim = C.c_uint64(), C.c_uint64()
        check(lib().parnn_replica_lowrank_state(self.h, layer, side, None, None, None, C.byref(rank), C.byref(dim)))
        w = np.zeros((rank.value, dim.value))
        d = np.zeros(rank.value)
        rho = C.c_double()
        check(lib().parnn_replica_lowrank_state(self.h, layer, side, ptr(w), ptr(d), C.byref(rho), None, None))
        return w, d, rho.value

    def lowrank_diag(self, layer: int, side: int) -> dict:
        out = np.zeros(6)
        check(lib().parnn_replica_lowrank_diag(self.h, layer, side, ptr(out)))
        return {"trxx": out[0], "gamma": out[1], "sweeps": int(out[2]), "jacobi_cycles": out[3],
                "eig_start_ns": out[4], "eig_end_ns": out[5]}

    def bind(self, ds: DeviceDataset):
        check(lib().parnn_replica_bind(self.h, ds.h))
        self.bound = ds

    def upload_epoch(self, rows, lrs):
        r = np.ascontiguousarray(rows, np.uint32).ravel()
        l = np.ascontiguousarray(lrs, np.float32)
        check(lib().parnn_replica_upload_epoch(self.h, ptr(r), ptr(l), l.size))

    def step(self, n: int = 1):
        check(lib().parnn_replica_step(self.h, n))

    def sync(self):
        check(lib().parnn_replica_sync(self.h))

    def ce(self, steps: int) -> np.ndarray:
        out = np.zeros(steps)
        check(lib().parnn_replica_ce(self.h, ptr(out), steps))
        return out

    def step_ce(self, step: int) -> float:
        """CE of one step of the epoch; waits for that step only."""
        out = C.c_double()
        check(lib().parnn_replica_step_ce(self.h, step, C.byref(out)))
        return out.value

    def forward(self, ds: DeviceDataset, rows) -> np.ndarray:
        r = np.ascontiguousarray(rows, np.uint32)
        z = np.zeros((r.size, self.dims[-1]), np.float32)
        check(lib().parnn_replica_forward(self.h, ds.h, ptr(r), r.size, ptr(z)))
        return z

    def accuracy(self, ds: DeviceDataset) -> float:
        out = C.c_double()
        check(lib().parnn_replica_accuracy(self.h, ds.h, C.byref(out)))
        return out.value

    def time_steps(self, steps: int) -> float:
        """Device ms (CUDA events on the replica stream) for `steps` graph launches."""
        out = C.c_double()
        check(lib().parnn_replica_time_steps(self.h, steps, C.byref(out)))
        return out.value

    def profile(self, steps: int = 1):
        """Eager profiled steps -> list of (region, avg ms, algorithmic flops)."""
        names = C.create_string_buffer(1 << 16)
        cap = 4096
        ms, fl = np.zeros(cap), np.zeros(cap)
        n = C.c_uint64()
        check(lib().parnn_replica_profile(self.h, steps, names, len(names), ptr(ms), ptr(fl), cap, C.byref(n)))
        labels = names.value.decode().split("\n")[:n.value]
        return [(labels[i], float(ms[i]), float(fl[i])) for i in range(n.value)]

    def kernels_per_step(self) -> int:
        out = C.c_uint64()
        check(lib().parnn_replica_kernels_per_step(self.h, C.byref(out)))
        return out.value

    def close(self):
        if self.h:
            lib().parnn_replica_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def average(replicas, comm=None, m_total: int | None = None) -> None:
    """allreduce_average over device replicas (+ NCCL comm across processes)."""
    arr = (C.c_void_p * len(replicas))(*[r.h for r in replicas])
    check(lib().parnn_average(arr, len(replicas), comm.h if comm else None,
                              m_total if m_total is not None else len(replicas)))


def run_steps(replicas, steps: int, avg_frequency: int, comm=None, m_total: int | None = None) -> float:
    """Device-timed inner loop of worker_epoch over local replicas (+ comm)."""
    arr = (C.c_void_p * len(replicas))(*[r.h for r in replicas])
    out = C.c_double()
    check(lib().parnn_run_steps(arr, len(replicas), comm.h if comm else None,
                                m_total if m_total is not None else len(replicas), steps, avg_frequency,
                                C.byref(out)))
    return out.value


def time_average(replicas, comm=None, m_total: int | None = None, iters: int = 10) -> tuple[float, float]:
    """Device ms per averaging event (CUDA events, back to back) and the fp32
    bytes one event reduces per GPU."""
    arr = (C.c_void_p * len(replicas))(*[r.h for r in replicas])
    ms, nb = C.c_double(), C.c_double()
    check(lib().parnn_time_average(arr, len(replicas), comm.h if comm else None,
                                   m_total if m_total is not None else len(replicas), iters, C.byref(ms),
                                   C.byref(nb)))
    return ms.value, nb.value


class Averager:
    """A persistent averaging group (allreduce_average over local replicas +
    comm): run() enqueues one averaging event without blocking the host."""

    def __init__(self, replicas, comm=None, m_total: int | None = None):
        arr = (C.c_void_p * len(replicas))(*[r.h for r in replicas])
        h = C.c_void_p()
        check(lib().parnn_averager_create(arr, len(replicas), comm.h if comm else None,
                                          m_total if m_total is not None else len(replicas), C.byref(h)))
        self.h, self._keep = h, list(replicas)

    def run(self):
        check(lib().parnn_averager_run(self.h))

    def close(self):
        if self.h:
            lib().parnn_averager_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """NCCL communicator; the unique id travels through torch.distributed (plumbing)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(lib().parnn_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        h = C.c_void_p()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        check(lib().parnn_comm_create(ctx.h, buf, nranks, rank, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().parnn_comm_destroy(self.h)
            self.h = None


# ------------------------------------------------------------ training
def _train(plan: ParallelPlan, model0: MlpModel, train: Dataset, cv: Dataset, opts: TrainOptions, serial: bool,
           device: int = 0, comm: Comm | None = None, rank0: int = 0, local_workers: int = 0,
           ctx: Context | None = None, device_data: tuple | None = None) -> TrainResult:
    ctx = ctx or Context(device)
    if device_data is not None:  # (train, cv) already resident on ctx's device (repeated runs, sweeps)
        tr, cvd = device_data
    else:
        tr = DeviceDataset(ctx, train)
        cvd = DeviceDataset(ctx, cv) if cv is not None and cv.size() > 0 else None
    cfg = TrainConfig(plan.workers, plan.avg_frequency, plan.minibatch, plan.base_seed, int(opts.optimizer),
                      int(opts.lr_schedule), opts.lr_init, opts.epochs, opts.ng_decay, opts.ng_smoothing,
                      int(opts.precision), int(model0.activation), rank0, local_workers, int(serial),
                      opts.ng_rank_in, opts.ng_rank_out, opts.ng_update_period, opts.ng_history,
                      opts.ng_update_lag)
    d = u64(model0.layer_dims)
    out = np.zeros(param_count(model0.layer_dims))
    met = np.zeros((max(opts.epochs, 1), 7))
    n = C.c_uint64()
    check(lib().parnn_train(ctx.h, comm.h if comm else None, C.byref(cfg), ptr(d), len(d), ptr(f64(model0.params)),
                            tr.h, cvd.h if cvd else None, ptr(out), ptr(met), C.byref(n)))
    ms = [EpochMetrics(int(r[0]), r[1], r[2], r[3], r[4], int(r[5]), int(r[6])) for r in met[:n.value]]
    return TrainResult(MlpModel(list(model0.layer_dims), model0.activation, out), ms, sum(m.wall_seconds for m in ms))


def train_parallel(plan: ParallelPlan, model0: MlpModel, train: Dataset, cv: Dataset, opts: TrainOptions,
                   **placement) -> TrainResult:
    """train_parallel (parallel.hpp:73-75). ``placement`` (device, comm, rank0,
    local_workers) spreads the m workers over processes/GPUs; ``ctx`` and
    ``device_data`` (DeviceDataset train / cv uploaded once) let repeated runs
    share a context and the resident data set."""
    return _train(plan, model0, train, cv, opts, False, **placement)


def serial_train(model0: MlpModel, train: Dataset, cv: Dataset, opts: TrainOptions, minibatch: int,
                 base_seed: int, **placement) -> TrainResult:
    """serial_train (parallel.hpp:79-81): one worker, averaging frequency 1."""
    return _train(ParallelPlan(1, 1, minibatch, base_seed), model0, train, cv, opts, True, **placement)


# ----------------------------------------------------------------- RBM
class Rbm:
    """RbmParams + CD-1 on the GPU (pretrain.hpp:14-60). Params packed as
    [W (h x v), v_bias, h_bias]."""

    def __init__(self, ctx: Context, visible: int, hidden: int, gaussian: bool, batch: int = 128,
                 precision: Precision = Precision.tf32):
        h = C.c_void_p()
        check(lib().parnn_rbm_create(ctx.h, visible, hidden, int(gaussian), batch, int(precision), C.byref(h)))
        self.h, self.v, self.hd = h, visible, hidden

    def set_params(self, p):
        p = f64(p)
        check(lib().parnn_rbm_set_params(self.h, ptr(p)))

    def get_params(self) -> np.ndarray:
        out = np.zeros(self.hd * self.v + self.v + self.hd)
        check(lib().parnn_rbm_get_params(self.h, ptr(out)))
        return out

    def cd1(self, batch, lr: float, sampling: str = "philox", seed: int = 0, counter: int = 0, uniforms=None):
        mode = {"philox": 0, "threshold": 1, "uniforms": 2}[sampling]
        b = f64(batch)
        u = f64(uniforms) if uniforms is not None else None
        check(lib().parnn_rbm_cd1(self.h, ptr(b), b.shape[0], lr, mode, seed, counter, ptr(u) if u is not None else None))

    def hidden_probs(self, x) -> np.ndarray:
        x = f64(x)
        out = np.zeros((x.shape[0], self.hd))
        check(lib().parnn_rbm_hidden_probs(self.h, ptr(x), x.shape[0], ptr(out)))
        return out

    def reconstruction_error(self, x) -> float:
        x = f64(x)
        out = C.c_double()
        check(lib().parnn_rbm_reconstruction_error(self.h, ptr(x), x.shape[0], C.byref(out)))
        return out.value

    def close(self):
        if self.h:
            lib().parnn_rbm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def greedy_pretrain(dims, data, opts: PretrainOptions = PretrainOptions(), activation=Activation.sigmoid,
                    seed: int = 0, precision: Precision = Precision.tf32, ctx: Context | None = None) -> MlpModel:
    """greedy_pretrain (pretrain.hpp:74-76) with a fresh Rng(seed)."""
    ctx = ctx or Context(0)
    d = u64(dims)
    x = f64(data)
    out = np.zeros(param_count(dims))
    check(lib().parnn_greedy_pretrain(ctx.h, ptr(d), len(d), ptr(x), x.shape[0], opts.epochs, opts.lr_gaussian,
                                      opts.lr_bernoulli, opts.batch_size, seed, int(precision), ptr(out)))
    return MlpModel(list(map(int, dims)), Activation(activation), out)


def pretrain_last_stats() -> dict:
    """Device time of the last greedy_pretrain's CD-1 epochs on this thread
    (CUDA events around each layer's epoch loop), step count and flop."""
    sec, steps, flop = C.c_double(), C.c_uint64(), C.c_double()
    check(lib().parnn_pretrain_last_stats(C.byref(sec), C.byref(steps), C.byref(flop)))
    return {"cd1_device_seconds": sec.value, "cd1_steps": steps.value, "cd1_flop": flop.value}


# ------------------------------------------------------------ test hooks
EPI = {"fwd_act": 0, "fwd_linear": 1, "grad": 2, "grad_sgd": 3, "actgrad": 4, "ema": 5, "axpy": 6, "sub": 7,
       "partial": 8, "resid": 9}


def debug_gemm(a, b, mode: str, precision: Precision, a_mn: bool = False, b_mn: bool = False, out=None, bias=None,
               aux=None, act: int = 0, ksplit: int = 1, force_bn: int = 0, force_mc: int = 0, lower: bool = False,
               bias_col: int = -1, alpha: float = 1.0, beta: float = 0.0, lr: float = 0.0) -> dict:
    """One production tcgen05 GEMM (parnn_debug_gemm): D[m, n] = sum_k A(m, k) B(n, k)
    with A given [M x K] (or [K x M] when a_mn) and B [N x K] (or [K x N] when
    b_mn), then the epilogue `mode`. Returns {out, out2, sums, mc, bn, ksplit,
    flags, grid}."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    M, K = (a.shape[1], a.shape[0]) if a_mn else a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    o = np.ascontiguousarray(out if out is not None else np.zeros((M, N)), np.float32).copy()
    o2 = np.zeros((M, N), np.float32) if bias_col < 0 else np.zeros(M, np.float32)
    bs = np.ascontiguousarray(bias, np.float32) if bias is not None else None
    ax = np.ascontiguousarray(aux, np.float32) if aux is not None else None
    sums = np.zeros(2)
    info = np.zeros(6, np.int32)
    check(lib().parnn_debug_gemm(int(precision), int(a_mn), int(b_mn), M, N, K, EPI[mode], act, ksplit, force_bn,
                                 force_mc, int(lower), bias_col, alpha, beta, lr, ptr(a), ptr(b),
                                 ptr(bs) if bs is not None else None, ptr(ax) if ax is not None else None, ptr(o),
                                 ptr(o2), ptr(sums), ptr(info)))
    return {"out": o, "out2": o2, "sums": sums, "mc": int(info[0]), "bn": int(info[1]), "ksplit": int(info[2]),
            "flags": int(info[3]), "grid": int(info[4])}
