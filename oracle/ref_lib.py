"""TEST INFRASTRUCTURE ONLY — ctypes binding of ``oracle/_ref/libparnn_ref.so``
(the unmodified reference compiled by ``oracle/Makefile`` + ``ref_capi.cpp``).

Used by tests (to pin the numpy restatement and to generate golden fixtures)
and by ``bench.py --impl reference`` / the ``cpu_baseline`` leg. Never used by
the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libparnn_ref.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")


def build(quiet: bool = True) -> bool:
    """Compile the reference oracle when its sources are present (this
    container); on the GPU box only the prebuilt .so is used."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(LIB_PATH)
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


class RefLib:
    def __init__(self, path: str = LIB_PATH):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_param_count.restype = C.c_uint64
        L.ref_accuracy.restype = C.c_double
        L.ref_exponential_lr.restype = C.c_double
        L.ref_reconstruction_error.restype = C.c_double
        L.ref_time_steps.restype = C.c_double
        L.ref_time_ng_precondition.restype = C.c_double

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    @staticmethod
    def _dims(dims):
        return np.ascontiguousarray(dims, dtype=np.uint64)

    def rng_u64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self._chk(self.lib.ref_rng_u64(C.c_uint64(seed), C.c_uint64(n), out.ctypes.data_as(C.c_void_p)))
        return out

    def rng_uniform(self, seed, n):
        out = np.zeros(n)
        self._chk(self.lib.ref_rng_uniform(C.c_uint64(seed), C.c_uint64(n), out.ctypes.data_as(C.c_void_p)))
        return out

    def rng_index(self, seed, bound, n):
        out = np.zeros(n, np.uint64)
        self._chk(self.lib.ref_rng_index(C.c_uint64(seed), C.c_uint64(bound), C.c_uint64(n),
                                         out.ctypes.data_as(C.c_void_p)))
        return out

    def rng_gaussian(self, seed, n, mean=0.0, sd=1.0):
        out = np.zeros(n)
        self._chk(self.lib.ref_rng_gaussian(C.c_uint64(seed), C.c_uint64(n), C.c_double(mean),
                                            C.c_double(sd), out.ctypes.data_as(C.c_void_p)))
        return out

    def shuffled_indices(self, n, seed):
        out = np.zeros(n, np.uint64)
        self._chk(self.lib.ref_shuffled_indices(C.c_uint64(n), C.c_uint64(seed), out.ctypes.data_as(C.c_void_p)))
        return out

    def partition_rows(self, n, m, seed):
        s = n // m
        out = np.zeros(m * s, np.uint64)
        self._chk(self.lib.ref_partition_rows(C.c_uint64(n), C.c_uint64(m), C.c_uint64(seed),
                                              out.ctypes.data_as(C.c_void_p)))
        return out.reshape(m, s)

    def minibatch_rows(self, n, b, seed):
        out = np.zeros((n // b) * b, np.uint64)
        self._chk(self.lib.ref_minibatch_rows(C.c_uint64(n), C.c_uint64(b), C.c_uint64(seed),
                                              out.ctypes.data_as(C.c_void_p)))
        return out.reshape(n // b, b)

    def make_data(self, classes, dim, per_class, sep, seed, cv_fraction=0.1, split_seed=0, standardize=True):
        n = classes * per_class
        ncv_max = n
        tx = np.zeros((n, dim)); ty = np.zeros(n, np.int32)
        cx = np.zeros((ncv_max, dim)); cy = np.zeros(ncv_max, np.int32)
        ntr = C.c_uint64(); ncv = C.c_uint64()
        self._chk(self.lib.ref_make_data(
            C.c_uint64(classes), C.c_uint64(dim), C.c_uint64(per_class), C.c_double(sep), C.c_uint64(seed),
            C.c_double(cv_fraction), C.c_uint64(split_seed), C.c_int(int(standardize)),
            tx.ctypes.data_as(C.c_void_p), ty.ctypes.data_as(C.c_void_p), C.byref(ntr),
            cx.ctypes.data_as(C.c_void_p), cy.ctypes.data_as(C.c_void_p), C.byref(ncv)))
        a, b = ntr.value, ncv.value
        return (tx[:a].copy(), ty[:a].copy()), (cx[:b].copy(), cy[:b].copy())

    def generate_synthetic(self, classes, dim, per_class, sep, seed):
        n = classes * per_class
        x = np.zeros((n, dim)); y = np.zeros(n, np.int32)
        self._chk(self.lib.ref_generate_synthetic(C.c_uint64(classes), C.c_uint64(dim), C.c_uint64(per_class),
                                                  C.c_double(sep), C.c_uint64(seed),
                                                  x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p)))
        return x, y

    def param_count(self, dims):
        d = self._dims(dims)
        return int(self.lib.ref_param_count(d.ctypes.data_as(C.c_void_p), C.c_int(len(d))))

    def init_random(self, dims, seed, act=0):
        d = self._dims(dims)
        p = np.zeros(self.param_count(dims))
        self._chk(self.lib.ref_init_random(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
                                           C.c_uint64(seed), p.ctypes.data_as(C.c_void_p)))
        return p

    def forward(self, dims, params, x, labels, act=0):
        d = self._dims(dims)
        B = x.shape[0]
        tot = sum(B * v for v in dims[1:])
        z = np.zeros(tot); a = np.zeros(tot); ce = C.c_double()
        x = np.ascontiguousarray(x, np.float64); labels = np.ascontiguousarray(labels, np.int32)
        self._chk(self.lib.ref_forward(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
                                       np.ascontiguousarray(params).ctypes.data_as(C.c_void_p),
                                       x.ctypes.data_as(C.c_void_p), C.c_uint64(B),
                                       labels.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p),
                                       a.ctypes.data_as(C.c_void_p), C.byref(ce)))
        zs, as_, pos = [], [], 0
        for v in dims[1:]:
            zs.append(z[pos:pos + B * v].reshape(B, v)); as_.append(a[pos:pos + B * v].reshape(B, v)); pos += B * v
        return zs, as_, ce.value

    def backward(self, dims, params, x, labels, act=0):
        d = self._dims(dims)
        B = x.shape[0]
        g = np.zeros(self.param_count(dims))
        dz = np.zeros(sum(B * v for v in dims[1:]))
        x = np.ascontiguousarray(x, np.float64); labels = np.ascontiguousarray(labels, np.int32)
        self._chk(self.lib.ref_backward(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
                                        np.ascontiguousarray(params).ctypes.data_as(C.c_void_p),
                                        x.ctypes.data_as(C.c_void_p), C.c_uint64(B),
                                        labels.ctypes.data_as(C.c_void_p), g.ctypes.data_as(C.c_void_p),
                                        dz.ctypes.data_as(C.c_void_p)))
        dzs, pos = [], 0
        for v in dims[1:]:
            dzs.append(dz[pos:pos + B * v].reshape(B, v)); pos += B * v
        return g, dzs

    def train_steps(self, dims, params0, x, labels, rows, batch, lrs, ngsgd, decay=0.95, smoothing=4.0, act=0):
        d = self._dims(dims)
        steps = len(lrs)
        rows = np.ascontiguousarray(rows, np.uint64).ravel()
        assert rows.size == steps * batch
        p = np.zeros(self.param_count(dims)); ce = np.zeros(steps)
        nf = sum(dims[l] ** 2 + dims[l + 1] ** 2 for l in range(len(dims) - 1))
        f = np.zeros(nf); g = np.zeros(self.param_count(dims))
        x = np.ascontiguousarray(x, np.float64); labels = np.ascontiguousarray(labels, np.int32)
        lrs = np.ascontiguousarray(lrs, np.float64)
        self._chk(self.lib.ref_train_steps(
            d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
            np.ascontiguousarray(params0).ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p),
            C.c_uint64(x.shape[0]), labels.ctypes.data_as(C.c_void_p), rows.ctypes.data_as(C.c_void_p),
            C.c_uint64(batch), C.c_uint64(steps), lrs.ctypes.data_as(C.c_void_p), C.c_int(int(ngsgd)),
            C.c_double(decay), C.c_double(smoothing), p.ctypes.data_as(C.c_void_p),
            ce.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p), g.ctypes.data_as(C.c_void_p)))
        factors, pos = [], 0
        for l in range(len(dims) - 1):
            a, b = dims[l], dims[l + 1]
            ri = f[pos:pos + a * a].reshape(a, a); pos += a * a
            ro = f[pos:pos + b * b].reshape(b, b); pos += b * b
            factors.append((ri, ro))
        return p, ce, factors, g

    def ng_precondition_layer(self, r_in, r_out, smoothing, gw, gb):
        do, di = gw.shape
        ow = np.zeros((do, di)); ob = np.zeros(do)
        args = [np.ascontiguousarray(v, np.float64) for v in (r_in, r_out, gw, gb)]
        self._chk(self.lib.ref_ng_precondition_layer(
            C.c_uint64(do), C.c_uint64(di), args[0].ctypes.data_as(C.c_void_p), args[1].ctypes.data_as(C.c_void_p),
            C.c_double(smoothing), args[2].ctypes.data_as(C.c_void_p), args[3].ctypes.data_as(C.c_void_p),
            ow.ctypes.data_as(C.c_void_p), ob.ctypes.data_as(C.c_void_p)))
        return ow, ob

    def allreduce_average(self, vs):
        vs = np.ascontiguousarray(vs, np.float64)
        m, n = vs.shape
        out = np.zeros(n)
        self._chk(self.lib.ref_allreduce_average(vs.ctypes.data_as(C.c_void_p), C.c_uint64(m), C.c_uint64(n),
                                                 out.ctypes.data_as(C.c_void_p)))
        return out

    def train_parallel(self, dims, params0, tx, ty, cx, cy, workers=1, avg_frequency=10, minibatch=128,
                       base_seed=0, ngsgd=True, newbob=False, lr_init=0.32, epochs=15, decay=0.95,
                       smoothing=4.0, serial=False, act=0):
        d = self._dims(dims)
        p = np.zeros(self.param_count(dims)); met = np.zeros((max(epochs, 1), 7)); n = C.c_uint64()
        arrs = [np.ascontiguousarray(v) for v in (tx.astype(np.float64), ty.astype(np.int32),
                                                   cx.astype(np.float64), cy.astype(np.int32))]
        self._chk(self.lib.ref_train_parallel(
            d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
            np.ascontiguousarray(params0).ctypes.data_as(C.c_void_p), arrs[0].ctypes.data_as(C.c_void_p),
            arrs[1].ctypes.data_as(C.c_void_p), C.c_uint64(tx.shape[0]), arrs[2].ctypes.data_as(C.c_void_p),
            arrs[3].ctypes.data_as(C.c_void_p), C.c_uint64(cx.shape[0]), C.c_uint64(workers),
            C.c_uint64(avg_frequency), C.c_uint64(minibatch), C.c_uint64(base_seed), C.c_int(int(ngsgd)),
            C.c_int(int(newbob)), C.c_double(lr_init), C.c_uint64(epochs), C.c_double(decay),
            C.c_double(smoothing), C.c_int(int(serial)), p.ctypes.data_as(C.c_void_p),
            met.ctypes.data_as(C.c_void_p), C.byref(n)))
        return p, met[:n.value]

    def accuracy(self, dims, params, x, y, act=0):
        d = self._dims(dims)
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.int32)
        return self.lib.ref_accuracy(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), C.c_int(act),
                                     np.ascontiguousarray(params).ctypes.data_as(C.c_void_p),
                                     x.ctypes.data_as(C.c_void_p), C.c_uint64(x.shape[0]),
                                     y.ctypes.data_as(C.c_void_p))

    def newbob_sequence(self, lr_init, accs):
        accs = np.ascontiguousarray(accs, np.float64)
        lr = np.zeros(len(accs) - 1); st = np.zeros(len(accs) - 1, np.int32)
        self._chk(self.lib.ref_newbob_sequence(C.c_double(lr_init), accs.ctypes.data_as(C.c_void_p),
                                               C.c_uint64(len(accs)), lr.ctypes.data_as(C.c_void_p),
                                               st.ctypes.data_as(C.c_void_p)))
        return lr, st

    def exponential_lr(self, lr_init, epochs, progress):
        return self.lib.ref_exponential_lr(C.c_double(lr_init), C.c_uint64(epochs), C.c_double(progress))

    def rbm_init(self, v, h, gaussian, seed):
        p = np.zeros(h * v + v + h)
        self._chk(self.lib.ref_rbm_init(C.c_uint64(v), C.c_uint64(h), C.c_int(int(gaussian)), C.c_uint64(seed),
                                        p.ctypes.data_as(C.c_void_p)))
        return p

    def cd1_update(self, v, h, gaussian, p, batch, lr, mode, seed=0):
        b = batch.shape[0]
        out = np.zeros_like(p); tr = np.zeros(b * h * 3 + b * v)
        batch = np.ascontiguousarray(batch, np.float64)
        self._chk(self.lib.ref_cd1_update(C.c_uint64(v), C.c_uint64(h), C.c_int(int(gaussian)),
                                          np.ascontiguousarray(p).ctypes.data_as(C.c_void_p),
                                          batch.ctypes.data_as(C.c_void_p), C.c_uint64(b), C.c_double(lr),
                                          C.c_int(mode), C.c_uint64(seed), out.ctypes.data_as(C.c_void_p),
                                          tr.ctypes.data_as(C.c_void_p)))
        pos = tr[:b * h].reshape(b, h); hs = tr[b * h:2 * b * h].reshape(b, h)
        rec = tr[2 * b * h:2 * b * h + b * v].reshape(b, v); neg = tr[2 * b * h + b * v:].reshape(b, h)
        return out, (pos, hs, rec, neg)

    def reconstruction_error(self, v, h, gaussian, p, batch):
        batch = np.ascontiguousarray(batch, np.float64)
        return self.lib.ref_reconstruction_error(C.c_uint64(v), C.c_uint64(h), C.c_int(int(gaussian)),
                                                 np.ascontiguousarray(p).ctypes.data_as(C.c_void_p),
                                                 batch.ctypes.data_as(C.c_void_p), C.c_uint64(batch.shape[0]))

    def greedy_pretrain(self, dims, data, epochs, lr_g, lr_b, batch, seed):
        d = self._dims(dims)
        p = np.zeros(self.param_count(dims))
        data = np.ascontiguousarray(data, np.float64)
        self._chk(self.lib.ref_greedy_pretrain(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)),
                                               data.ctypes.data_as(C.c_void_p), C.c_uint64(data.shape[0]),
                                               C.c_uint64(epochs), C.c_double(lr_g), C.c_double(lr_b),
                                               C.c_uint64(batch), C.c_uint64(seed), p.ctypes.data_as(C.c_void_p)))
        return p

    def save_model(self, path, dims, params, act=0):
        d = self._dims(dims)
        self._chk(self.lib.ref_save_model(path.encode(), d.ctypes.data_as(C.c_void_p), C.c_int(len(d)),
                                          C.c_int(act), np.ascontiguousarray(params).ctypes.data_as(C.c_void_p)))

    def time_steps(self, dims, params, x, y, batch, steps, ngsgd, threads):
        d = self._dims(dims)
        ph = np.zeros(5)
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.int32)
        fps = self.lib.ref_time_steps(d.ctypes.data_as(C.c_void_p), C.c_int(len(d)),
                                      np.ascontiguousarray(params).ctypes.data_as(C.c_void_p),
                                      x.ctypes.data_as(C.c_void_p), C.c_uint64(x.shape[0]),
                                      y.ctypes.data_as(C.c_void_p), C.c_uint64(batch), C.c_uint64(steps),
                                      C.c_int(int(ngsgd)), C.c_int(threads), ph.ctypes.data_as(C.c_void_p))
        if fps < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return fps, ph

    def time_ng_precondition(self, d_out, d_in, batch=64, seed=1):
        s = self.lib.ref_time_ng_precondition(C.c_uint64(d_out), C.c_uint64(d_in), C.c_uint64(batch),
                                              C.c_uint64(seed))
        if s < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return s

    def time_step_threaded(self, dims, params, x, labels, ngsgd, threads, lr=1e-3):
        """One true-width minibatch step of the reference (worker_epoch's body)
        from its own public functions on `threads` host threads
        (ref_time_step_threaded). Returns (wall seconds, phase seconds[7],
        params after the step, batch CE)."""
        d = self._dims(dims)
        x = np.ascontiguousarray(x, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        ph = np.zeros(7)
        p = np.zeros(self.param_count(dims))
        ce = C.c_double()
        self.lib.ref_time_step_threaded.restype = C.c_double
        wall = self.lib.ref_time_step_threaded(
            d.ctypes.data_as(C.c_void_p), C.c_int(len(d)), np.ascontiguousarray(params).ctypes.data_as(C.c_void_p),
            x.ctypes.data_as(C.c_void_p), labels.ctypes.data_as(C.c_void_p), C.c_uint64(x.shape[0]),
            C.c_int(int(ngsgd)), C.c_int(threads), C.c_double(lr), ph.ctypes.data_as(C.c_void_p),
            p.ctypes.data_as(C.c_void_p), C.byref(ce))
        if wall < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return wall, ph, p, ce.value

    def load_csv(self, path):
        """The reference's load_csv: (x, y, classes); raises RuntimeError with its message."""
        n, d, k = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._chk(self.lib.ref_load_csv(path.encode(), None, None, C.c_uint64(0), C.c_uint64(0), C.byref(n),
                                        C.byref(d), C.byref(k)))
        x = np.zeros((n.value, d.value)); y = np.zeros(n.value, np.int32)
        self._chk(self.lib.ref_load_csv(path.encode(), x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p),
                                        C.c_uint64(n.value), C.c_uint64(d.value), C.byref(n), C.byref(d),
                                        C.byref(k)))
        return x, y, k.value

    def save_csv(self, path, x, y):
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.int32)
        self._chk(self.lib.ref_save_csv(path.encode(), x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p),
                                        C.c_uint64(x.shape[0]), C.c_uint64(x.shape[1])))
