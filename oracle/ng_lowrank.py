"""TEST INFRASTRUCTURE ONLY — CPU restatement (numpy, fp64) of the low-rank
online natural-gradient preconditioner.

PARITY UNPINNED. The reference (/root/reference/proj) does not implement this
algorithm; it is the north star's NG-SGD ("per-layer low-rank Fisher
projection and rank-R subspace update"). This module restates the published
algorithm of Povey, Zhang & Khudanpur, "Parallel training of DNNs with natural
gradient and parameter averaging" (arXiv:1410.7455, 2014), section 3 and
appendix C ("online" NG-SGD). It is the only oracle for A17: the GPU
implementation (paper_1507_01239_b200/csrc/ng_lowrank.cu) is checked against
it in fp32 mode, and the low-rank trainer as a whole is checked statistically
against the reference's kron-full NG-SGD (final CE), as SURVEY §8a/A17 asks.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may import it.

Notation (per layer, per side): X is N x D (side "in": [A_prev | 1], the
input activations with the bias column appended; side "out": the per-example
output derivatives dz, no 1/N). The Fisher estimate is
    F_t = R_t^T D_t R_t + rho_t I          (R_t: R x D, orthonormal rows)
stored as W_t = E_t^{1/2} R_t with E_t = diag(e_i), e_i = d_i / (d_i + beta_t),
    beta_t = rho_t (1 + alpha) + alpha tr(D_t) / D.
Preconditioning (X F~^-1 up to scale, F~ = F + alpha tr(F)/D I):
    H = X W^T,  X^ = X - H W,  gamma = sqrt(tr(X X^T) / tr(X^ X^T)).
Subspace update every `update_period` calls (eta = 1 - exp(-N P / S)), in
effect update_lag calls later (1 = the next call, as in the paper; the default
here is 4 = the update period, which lets the device overlap the eigensolve
with the three steps in between):
    T = (eta/N) X^T X + (1 - eta) F_t,    Y = R_t T,   Z = Y Y^T = U C^2 U^T
    R_{t+1} = C^-1 U^T Y,  rho_{t+1} = (tr T - tr C) / (D - R),  D_{t+1} = C - rho_{t+1}
with the floors c, d >= max(DELTA c_max, EPS tr(T)/D) and rho >= EPS tr(T)/D
(scale-relative, so the update is invariant to the scale of X and stays
bounded for rank-deficient X, where R_{t+1} rows of floored directions
shrink instead of blowing up), and Y and Z formed from J = H^T X (R x D) and the R x R Gram blocks
K = J J^T, L = W J^T (= H^T H) and G = W W^T, so nothing D x D is ever built.
The first call runs `init_iters` updates on its own batch from a fixed
orthonormal basis (lowrank_basis) before preconditioning.

The layer gradient is formed from the preconditioned vectors:
    gW = gamma_in gamma_out / N  D^^T A^[:, :din],
    gb = gamma_in gamma_out / N  D^^T A^[:, din]   (the preconditioned ones column)
then the reference's sgd_step (optimizer.cpp:9-36) applies it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .parnn_oracle import Model, Rng, backward, cross_entropy, forward, sgd_step

EPS = 1e-10    # floor of rho relative to the mean eigenvalue tr(T)/D
DELTA = 5e-4   # floor of c and d relative to the largest c (bounds C^-1: rank-deficient inputs)
TINY = 1e-30


@dataclass
class LowRankConfig:
    rank_in: int = 20
    rank_out: int = 80
    update_period: int = 4
    num_samples_history: float = 2000.0
    alpha: float = 4.0
    init_iters: int = 3
    update_lag: int = 4  # steps until an update computed at step t takes effect (1 = t+1 as in Kaldi; <= P)


def basis_seed(layer: int, side: int) -> int:
    """Seed of the initial basis of (layer, side); side 0 = in, 1 = out."""
    return 0x4C52_4E47_0000 + 2 * layer + side


def effective_rank(rank: int, dim: int) -> int:
    return max(1, min(rank, dim - 1))


def lowrank_basis(dim: int, rank: int, seed: int) -> np.ndarray:
    """rank x dim matrix with orthonormal rows: Rng(seed).gaussian(0, 1) drawn
    row-major, then modified Gram-Schmidt in fp64 (host.cpp lowrank_basis)."""
    rng = Rng(seed)
    m = np.empty((rank, dim))
    for i in range(rank):
        for j in range(dim):
            m[i, j] = rng.gaussian(0.0, 1.0)
    for i in range(rank):
        v = m[i]
        for k in range(i):
            v = v - float(np.dot(m[k], v)) * m[k]
        m[i] = v / math.sqrt(float(np.dot(v, v)))
    return m


def e_of(d, rho, dim, alpha):
    beta = rho * (1.0 + alpha) + alpha * float(d.sum()) / dim
    return d / (d + beta)


@dataclass
class Side:
    dim: int
    rank: int
    W: np.ndarray
    d: np.ndarray
    rho: float
    e: np.ndarray
    t: int = 0
    pending: tuple = None  # (W, d, rho, e) of an update computed but not yet in effect
    pending_due: int = 0


def side_init(dim: int, rank: int, seed: int, alpha: float) -> Side:
    r = effective_rank(rank, dim)
    d = np.full(r, EPS)
    rho = EPS
    e = e_of(d, rho, dim, alpha)
    return Side(dim, r, np.sqrt(e)[:, None] * lowrank_basis(dim, r, seed), d, rho, e)


def precondition(st: Side, x):
    """H, X^, gamma, tr(X X^T)."""
    h = x @ st.W.T
    xh = x - h @ st.W
    trxx = float((x * x).sum())
    trhh = float((xh * xh).sum())
    gamma = math.sqrt(trxx / trhh) if trhh > 0.0 else 1.0
    return h, xh, gamma, trxx


def eig_update(d, e, rho, K, L, G, trxx, D, eta, a, alpha):
    """The R x R part of the subspace update: (d', rho', e', M) with
    W' = M [J; W] = [M1 | M2] [J; W] (ng_lowrank.cu lr_eig_kernel)."""
    R = d.shape[0]
    dr = d + rho
    zi = a * a * K + a * (1.0 - eta) * (L * dr[None, :] + dr[:, None] * L) \
        + (1.0 - eta) ** 2 * (dr[:, None] * G * dr[None, :])
    ih = 1.0 / np.sqrt(e)
    z = ih[:, None] * zi * ih[None, :]
    z = 0.5 * (z + z.T)
    lam, u = np.linalg.eigh(z)
    order = np.argsort(-lam, kind="stable")
    lam, u = lam[order], u[:, order]
    trt = a * trxx + (1.0 - eta) * (D * rho + float(d.sum()))
    c = np.sqrt(np.maximum(lam, 0.0))
    floor = max(DELTA * float(c.max()), EPS * trt / D, TINY)  # scale-relative floors
    c = np.maximum(c, floor)
    rho1 = max((trt - float(c.sum())) / (D - R), EPS * trt / D, TINY)
    d1 = np.maximum(c - rho1, floor)
    e1 = e_of(d1, rho1, D, alpha)
    m = (np.sqrt(e1) / c)[:, None] * u.T * ih[None, :]
    return d1, rho1, e1, np.concatenate([a * m, (1.0 - eta) * m * dr[None, :]], axis=1)


def compute_update(st: Side, x, h, trxx: float, eta: float, alpha: float):
    n = x.shape[0]
    j = h.T @ x
    a = eta / n
    d1, rho1, e1, m = eig_update(st.d, st.e, st.rho, j @ j.T, st.W @ j.T, st.W @ st.W.T, trxx, st.dim, eta, a,
                                 alpha)
    return m @ np.concatenate([j, st.W], axis=0), d1, rho1, e1


def update(st: Side, x, h, trxx: float, eta: float, alpha: float) -> None:
    st.W, st.d, st.rho, st.e = compute_update(st, x, h, trxx, eta, alpha)


def eta_of(n: int, cfg: LowRankConfig) -> float:
    return 1.0 - math.exp(-n * cfg.update_period / cfg.num_samples_history)


def effective_lag(cfg: LowRankConfig) -> int:
    """An update must take effect before the next one is computed: lag <= P."""
    return max(1, min(cfg.update_lag, cfg.update_period))


def side_step(st: Side, x, cfg: LowRankConfig):
    """One preconditioning call: init on the first call, precondition with
    W_t, then update the subspace every update_period calls. The update
    computed from call t takes effect at call t + update_lag (lag >= 2: the
    device computes it in the background during the calls in between)."""
    eta = eta_of(x.shape[0], cfg)
    if st.t == 0:
        for _ in range(cfg.init_iters):
            h, _, _, trxx = precondition(st, x)
            update(st, x, h, trxx, eta, cfg.alpha)
    if st.pending is not None and st.t >= st.pending_due:
        st.W, st.d, st.rho, st.e = st.pending
        st.pending = None
    h, xh, gamma, trxx = precondition(st, x)
    if st.t % cfg.update_period == 0:
        if effective_lag(cfg) == 1:
            update(st, x, h, trxx, eta, cfg.alpha)
        else:
            st.pending = compute_update(st, x, h, trxx, eta, cfg.alpha)
            st.pending_due = st.t + effective_lag(cfg)
    st.t += 1
    return xh, gamma


@dataclass
class LowRankState:
    cfg: LowRankConfig
    sides_in: list = field(default_factory=list)
    sides_out: list = field(default_factory=list)


def lowrank_init(m: Model, cfg: LowRankConfig | None = None) -> LowRankState:
    cfg = cfg or LowRankConfig()
    st = LowRankState(cfg)
    for l in range(len(m.W)):
        din, dout = m.dims[l], m.dims[l + 1]
        st.sides_in.append(side_init(din + 1, cfg.rank_in, basis_seed(l, 0), cfg.alpha))
        st.sides_out.append(side_init(dout, cfg.rank_out, basis_seed(l, 1), cfg.alpha))
    return st


def lowrank_gradients(st: LowRankState, m: Model, tr, dzs):
    """Preconditioned (gW, gb) per layer from the trace and per-example dz."""
    n = tr.x.shape[0]
    gW, gb = [], []
    for l in range(len(m.W)):
        a = tr.x if l == 0 else tr.a[l - 1]
        xin = np.concatenate([a, np.ones((n, 1))], axis=1)
        ah, g_in = side_step(st.sides_in[l], xin, st.cfg)
        dh, g_out = side_step(st.sides_out[l], dzs[l], st.cfg)
        s = g_in * g_out / n
        gW.append(s * (dh.T @ ah[:, :-1]))
        gb.append(s * (dh.T @ ah[:, -1]))
    return gW, gb


def lowrank_train_steps(m: Model, st: LowRankState, x, y, batches, lrs):
    """`len(batches)` minibatch updates (forward, CE, backward, low-rank NG,
    sgd_step); returns the per-step CE. Mutates m and st."""
    ces = []
    for rows, lr in zip(batches, lrs):
        tr = forward(m, x[rows])
        ces.append(cross_entropy(tr, y[rows]))
        _, _, dzs = backward(m, tr, y[rows], want_dz=True)
        gW, gb = lowrank_gradients(st, m, tr, dzs)
        sgd_step(m, gW, gb, lr)
    return ces
