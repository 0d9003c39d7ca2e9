"""NumPy restatement of the reference GSpaRC renderer / trainer (the oracle).

TEST INFRASTRUCTURE -- not product code.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (CPU-baseline leg and the
`--impl reference` arm) may import it.  The CUDA product path never calls it.

Every function cites the reference file:line it restates; paths are relative
to `/root/reference/pkg/src/rfsplat/`.  Parity of this restatement with the
reference itself is pinned by `tests/test_oracle_golden.py` against fixtures
written by `tests/golden/make_golden.py`, which imports the real reference.

Generalisations beyond the reference (documented, validated by linearity in
the golden generator):
  * `C = mlp_out` channels instead of the hard-coded 2
    (`rasterizer.py:192,216,243,258,277,280`), so one call renders all
    F subcarriers (C = 2F);
  * batched transmitters are a loop over `forward`.

Arrays are plain float64 NumPy arrays in the reference's parameter layout
(`scene.py:46-103`): pos (N,3), log_scales (N,3), rotations (N,4) as
(w,x,y,z), raw_opacities (N,1), mlp_weights (N,P) with rows
W1(h x i) | b1(h) | W2(o x h) | b2(o)  (`mlp.py:6-7`).
"""

from __future__ import annotations

import math
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------- constants
# rasterizer.py:33-36, geometry.py:19-31, scene.py:19-22, optimize.py:20-24
ALPHA_MAX = 0.99
ALPHA_MIN = 1.0 / 255.0
T_EPS = 1e-4
TILE = 16
COV2D_REG = 0.3
FOOTPRINT_SIGMA = float(np.sqrt(2.0 * np.log(255.0)))
NEAR_PLANE = 0.05
FAR_PLANE = 1000.0
POLE_CLAMP_DEG = 89.0
DEFAULT_MLP_DIMS = (5, 16, 2)
SSIM_WIN, SSIM_SIG, SSIM_K1, SSIM_K2 = 11, 1.5, 0.01, 0.03
GROUPS = ("positions", "log_scales", "rotations", "raw_opacities",
          "mlp_weights")


def n_mlp_params(dims):
    """scene.py:25-27."""
    i, h, o = dims
    return i * h + h + h * o + o


@dataclass
class Cloud:
    """Plain f64 parameter arrays (scene.py:46-103)."""

    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    raw_opacities: np.ndarray
    mlp_weights: np.ndarray
    mlp_dims: tuple = DEFAULT_MLP_DIMS

    @property
    def n(self):
        return self.positions.shape[0]

    def groups(self):
        return {g: getattr(self, g) for g in GROUPS}

    def copy(self):
        return Cloud(*(getattr(self, g).copy() for g in GROUPS),
                     mlp_dims=tuple(self.mlp_dims))


def as_cloud(obj):
    """Accept any object with the reference's five arrays + mlp_dims."""
    if isinstance(obj, Cloud):
        return obj
    arrs = [np.asarray(getattr(obj, g), dtype=np.float64) for g in GROUPS]
    return Cloud(*arrs, mlp_dims=tuple(getattr(obj, "mlp_dims",
                                               DEFAULT_MLP_DIMS)))


# ------------------------------------------------------------ activations
def sigmoid(raw):
    """Split-branch stable sigmoid (scene.py:106-114)."""
    raw = np.asarray(raw, dtype=np.float64)
    out = np.empty_like(raw)
    p = raw >= 0
    out[p] = 1.0 / (1.0 + np.exp(-raw[p]))
    e = np.exp(raw[~p])
    out[~p] = e / (1.0 + e)
    return out


def unit_quat(q):
    """scene.py:117-122."""
    q = np.asarray(q, dtype=np.float64)
    nrm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(nrm == 0.0):
        raise ValueError("zero quaternion")
    return q / nrm


def quat_to_rot(q):
    """(w,x,y,z) -> R (scene.py:125-139)."""
    w, x, y, z = (q[..., k] for k in range(4))
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def covariance3d(cloud: Cloud):
    """Sigma = (R diag e^s)(R diag e^s)^T (scene.py:84-88)."""
    M = quat_to_rot(unit_quat(cloud.rotations)) * \
        np.exp(cloud.log_scales)[:, None, :]
    return M @ np.swapaxes(M, 1, 2)


def quat_grad(q_raw, g_R):
    """Gradient through R(normalize(q)) (scene.py:142-173)."""
    qh = unit_quat(q_raw)
    w, x, y, z = (qh[..., k] for k in range(4))
    # dR/dw, dR/dx, dR/dy, dR/dz contracted with g_R, written out per entry
    G = g_R
    gw = 2 * (-z * G[..., 0, 1] + y * G[..., 0, 2] + z * G[..., 1, 0]
              - x * G[..., 1, 2] - y * G[..., 2, 0] + x * G[..., 2, 1])
    gx = 2 * (y * G[..., 0, 1] + z * G[..., 0, 2] + y * G[..., 1, 0]
              - 2 * x * G[..., 1, 1] - w * G[..., 1, 2] + z * G[..., 2, 0]
              + w * G[..., 2, 1] - 2 * x * G[..., 2, 2])
    gy = 2 * (-2 * y * G[..., 0, 0] + x * G[..., 0, 1] + w * G[..., 0, 2]
              + x * G[..., 1, 0] + z * G[..., 1, 2] - w * G[..., 2, 0]
              + z * G[..., 2, 1] - 2 * y * G[..., 2, 2])
    gz = 2 * (-2 * z * G[..., 0, 0] - w * G[..., 0, 1] + x * G[..., 0, 2]
              + w * G[..., 1, 0] - 2 * z * G[..., 1, 1] + y * G[..., 1, 2]
              + x * G[..., 2, 0] + y * G[..., 2, 1])
    gh = np.stack([gw, gx, gy, gz], -1)
    nrm = np.linalg.norm(q_raw, axis=-1, keepdims=True)
    return (gh - qh * np.sum(gh * qh, axis=-1, keepdims=True)) / nrm


# ---------------------------------------------------------------- geometry
def to_view(pos, rx, W):
    """W (mu - x_rx) (geometry.py:61-64)."""
    return (np.asarray(pos, np.float64) - rx) @ W.T


def project(p, w, h):
    """Equirect pixel coords (geometry.py:67-80)."""
    x, y, z = p[..., 0], p[..., 1], p[..., 2]
    r = np.sqrt(x * x + y * y + z * z)
    px = (np.arctan2(x, z) / np.pi + 1.0) * (w / 2.0)
    py = 2.0 * np.arcsin(np.clip(y / r, -1.0, 1.0)) * (h / np.pi)
    return np.stack([px, py], axis=-1)


def _pole_pull(p):
    """Move points above 89 deg elevation onto it (geometry.py:98-113)."""
    p = np.array(p, dtype=np.float64)
    x, y, z = p[..., 0], p[..., 1], p[..., 2]
    r = np.sqrt(x * x + y * y + z * z)
    lim = np.deg2rad(POLE_CLAMP_DEG)
    over = np.arcsin(np.clip(y / r, -1.0, 1.0)) > lim
    if np.any(over):
        az = np.arctan2(x, z)
        rho_t = r * np.cos(lim)
        nx = np.where(over, rho_t * np.sin(az), x)
        ny = np.where(over, r * np.sin(lim), y)
        nz = np.where(over, rho_t * np.cos(az), z)
        p[..., 0], p[..., 1], p[..., 2] = nx, ny, nz
    return p


def jacobian(p, w, h):
    """2x3 projection Jacobian with the pole clamp (geometry.py:116-149)."""
    p = np.atleast_2d(np.asarray(p, np.float64))
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    r2 = x * x + y * y + z * z
    rho2 = x * x + z * z
    lim = np.deg2rad(POLE_CLAMP_DEG)
    if np.any((rho2 <= r2 * np.cos(lim) ** 2) & (y > 0)):
        p = _pole_pull(p)
        x, y, z = p[:, 0], p[:, 1], p[:, 2]
        r2 = x * x + y * y + z * z
        rho2 = x * x + z * z
    rho = np.sqrt(rho2)
    ca = w / (2.0 * np.pi)
    ce = 2.0 * h / np.pi
    J = np.zeros((p.shape[0], 2, 3))
    J[:, 0, 0] = ca * z / rho2
    J[:, 0, 2] = -ca * x / rho2
    J[:, 1, 0] = -ce * x * y / (r2 * rho)
    J[:, 1, 1] = ce * rho / r2
    J[:, 1, 2] = -ce * y * z / (r2 * rho)
    return J


def jacobian_hessian(p, w, h):
    """d^2 P_k / dp_i dp_j, shape (M,2,3,3) (geometry.py:152-180)."""
    p = np.atleast_2d(_pole_pull(p))
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    rho2 = x * x + z * z
    rho = np.sqrt(rho2)
    r2 = rho2 + y * y
    r4 = r2 * r2
    ca = w / (2.0 * np.pi)
    ce = 2.0 * h / np.pi
    H = np.zeros((p.shape[0], 2, 3, 3))
    H[:, 0, 0, 0] = ca * (-2.0 * x * z / rho2 ** 2)
    H[:, 0, 0, 2] = H[:, 0, 2, 0] = ca * (x * x - z * z) / rho2 ** 2
    H[:, 0, 2, 2] = ca * (2.0 * x * z / rho2 ** 2)
    A = 2.0 / (r4 * rho) + 1.0 / (r2 * rho ** 3)
    H[:, 1, 0, 0] = ce * (-y / (r2 * rho) + x * x * y * A)
    H[:, 1, 0, 1] = H[:, 1, 1, 0] = ce * (-x * (r2 - 2.0 * y * y) / (r4 * rho))
    H[:, 1, 0, 2] = H[:, 1, 2, 0] = ce * (x * y * z * A)
    H[:, 1, 1, 1] = ce * (-2.0 * rho * y / r4)
    H[:, 1, 1, 2] = H[:, 1, 2, 1] = ce * (z * (y * y - rho2) / (rho * r4))
    H[:, 1, 2, 2] = ce * (-y / (r2 * rho) + z * z * y * A)
    return H


def _screen_cov(J, W, cov3d):
    """J W Sigma W^T J^T, same contraction as geometry.py:219-220 /
    rasterizer.py:92."""
    return np.einsum("nij,jk,nkl,ml,nom->nio", J, W, cov3d, W, J)


def visible_set(cloud: Cloud, rx, W, w, h):
    """Ascending indices kept by the view cull (geometry.py:198-224)."""
    mu = to_view(cloud.positions, rx, W)
    depth = np.linalg.norm(mu, axis=1)
    keep = (depth >= NEAR_PLANE) & (depth <= FAR_PLANE)
    with np.errstate(invalid="ignore", divide="ignore"):
        el = np.degrees(np.arcsin(np.clip(
            mu[:, 1] / np.maximum(depth, 1e-30), -1, 1)))
    keep &= el >= -90.0
    cand = np.nonzero(keep)[0]
    if cand.size == 0:
        return cand
    py = project(mu[cand], w, h)[:, 1]
    cov = _screen_cov(jacobian(mu[cand], w, h), W,
                      covariance3d(cloud)[cand]) + COV2D_REG * np.eye(2)
    ry = FOOTPRINT_SIGMA * np.sqrt(np.maximum(cov[:, 1, 1], 0.0))
    ok = (py + ry >= 0.0) & (py - ry <= float(h))
    return cand[ok]


# ---------------------------------------------------------------- MLP
def mlp_split(weights, dims):
    """Flat rows -> W1 (M,h,i), b1, W2 (M,o,h), b2 (mlp.py:17-30)."""
    i, h, o = dims
    weights = np.asarray(weights, np.float64)
    if weights.shape[-1] != n_mlp_params(dims):
        raise ValueError("MLP weight length mismatch")
    a = i * h
    W1 = weights[:, :a].reshape(-1, h, i)
    b1 = weights[:, a:a + h]
    W2 = weights[:, a + h:a + h + o * h].reshape(-1, o, h)
    b2 = weights[:, a + h + o * h:]
    return W1, b1, W2, b2


def mlp_fwd(weights, x, dims):
    """(mlp.py:40-45)."""
    W1, b1, W2, b2 = mlp_split(weights, dims)
    hid = np.maximum(np.einsum("mhi,mi->mh", W1, x) + b1, 0.0)
    return np.einsum("moh,mh->mo", W2, hid) + b2


def mlp_bwd(weights, x, up, dims):
    """(grad_w, grad_x) of mlp_fwd (mlp.py:48-70)."""
    i, h, o = dims
    W1, b1, W2, b2 = mlp_split(weights, dims)
    pre = np.einsum("mhi,mi->mh", W1, x) + b1
    hid = np.maximum(pre, 0.0)
    g_hid = np.einsum("moh,mo->mh", W2, up)
    g_pre = g_hid * (pre > 0.0)
    m = weights.shape[0]
    g_w = np.concatenate([
        (g_pre[:, :, None] * x[:, None, :]).reshape(m, h * i), g_pre,
        (up[:, :, None] * hid[:, None, :]).reshape(m, o * h), up], axis=1)
    return g_w, np.einsum("mhi,mh->mi", W1, g_pre)


def view_angles(mu):
    """(theta, phi) (mlp.py:83-89)."""
    x, y, z = mu[:, 0], mu[:, 1], mu[:, 2]
    return np.arctan2(x, z), np.arctan2(y, np.sqrt(x * x + z * z))


def view_angles_grad(mu, g_t, g_p):
    """(mlp.py:92-103)."""
    x, y, z = mu[:, 0], mu[:, 1], mu[:, 2]
    rho2 = x * x + z * z
    rho = np.sqrt(rho2)
    r2 = rho2 + y * y
    out = np.zeros_like(mu)
    out[:, 0] = g_t * (z / rho2) + g_p * (-x * y / (r2 * rho))
    out[:, 1] = g_p * (rho / r2)
    out[:, 2] = g_t * (-x / rho2) + g_p * (-y * z / (r2 * rho))
    return out


# ------------------------------------------------------- per-render state
@dataclass
class Prep:
    """Culled, depth-sorted per-Gaussian state (rasterizer.py:69-112)."""

    idx: np.ndarray
    w: int
    h: int
    mu_v: np.ndarray = None
    depth: np.ndarray = None
    mean2d: np.ndarray = None
    cov2d: np.ndarray = None
    conic: np.ndarray = None
    radii: np.ndarray = None
    opac: np.ndarray = None
    d_tx: np.ndarray = None
    d_clamped: np.ndarray = None
    inputs: np.ndarray = None
    s: np.ndarray = None
    J: np.ndarray = None


def prepare(cloud: Cloud, rx, W, tx, w, h):
    """Cull, depth sort (np.lexsort ties -> source index), projection,
    conic, radii, opacity, 1/d clamp and MLP (rasterizer.py:75-112)."""
    tx = np.asarray(tx, np.float64).reshape(3)
    keep = visible_set(cloud, rx, W, w, h)
    pr = Prep(idx=keep, w=int(w), h=int(h))
    if keep.size == 0:
        return pr
    mu = to_view(cloud.positions[keep], rx, W)
    depth = np.linalg.norm(mu, axis=1)
    order = np.lexsort((keep, depth))
    pr.idx = keep[order]
    pr.mu_v = mu[order]
    pr.depth = depth[order]
    pr.mean2d = project(pr.mu_v, w, h)
    pr.J = jacobian(pr.mu_v, w, h)
    c2 = _screen_cov(pr.J, W, covariance3d(cloud)[pr.idx])
    c2 = 0.5 * (c2 + np.swapaxes(c2, 1, 2))
    c2[:, 0, 0] += COV2D_REG
    c2[:, 1, 1] += COV2D_REG
    pr.cov2d = c2
    a, b, c = c2[:, 0, 0], c2[:, 0, 1], c2[:, 1, 1]
    det = a * c - b * b
    pr.conic = np.stack([c / det, -b / det, a / det], axis=1)
    pr.radii = FOOTPRINT_SIGMA * np.sqrt(np.stack([a, c], axis=1))
    pr.opac = sigmoid(cloud.raw_opacities[pr.idx, 0])
    d = np.linalg.norm(cloud.positions[pr.idx] - tx, axis=1)
    pr.d_clamped = d < NEAR_PLANE
    pr.d_tx = np.maximum(d, NEAR_PLANE)
    th, ph = view_angles(pr.mu_v)
    m = pr.idx.size
    pr.inputs = np.concatenate([np.broadcast_to(tx, (m, 3)), th[:, None],
                                ph[:, None]], axis=1)
    pr.s = mlp_fwd(cloud.mlp_weights[pr.idx], pr.inputs, cloud.mlp_dims)
    return pr


def tile_grid(w, h):
    return (w + TILE - 1) // TILE, (h + TILE - 1) // TILE


def tile_bins(pr: Prep):
    """Per-tile contributor rows in depth order, including the azimuth-seam
    duplicate quirk (rasterizer.py:115-145), computed without a Python loop
    over Gaussians.  Returns {(ty, tx): int array of rows}."""
    w, h = pr.w, pr.h
    ntx, nty = tile_grid(w, h)
    m = pr.idx.size
    if m == 0:
        return {}
    mx, my = pr.mean2d[:, 0], pr.mean2d[:, 1]
    rx, ry = pr.radii[:, 0], pr.radii[:, 1]
    ylo = np.clip(np.floor((my - ry - 0.5) / TILE).astype(int), 0, nty - 1)
    yhi = np.clip(np.floor((my + ry + 0.5) / TILE).astype(int), 0, nty - 1)
    vis = (my + ry >= 0.0) & (my - ry <= h)
    lo = np.mod(mx - rx - 0.5, w)
    span = 2.0 * rx + 1.0
    hi = lo + span
    full = span >= w
    wrap = (~full) & (hi >= w)
    # column segments [a0, a1] and (wrapped) [b0, b1]; b0 > b1 means empty
    a0 = np.where(full, 0, np.floor_divide(lo, TILE)).astype(int)
    a1 = np.where(full, ntx - 1,
                  np.where(wrap, ntx - 1, np.floor_divide(hi, TILE))).astype(int)
    b0 = np.zeros(m, int)
    b1 = np.where(wrap, np.floor_divide(hi - w, TILE), -1).astype(int)
    b1[~wrap] = -1
    rows, keys = [], []
    for ty in range(nty):
        iny = vis & (ylo <= ty) & (yhi >= ty)
        for tx_ in range(ntx):
            mult = (iny & (a0 <= tx_) & (a1 >= tx_)).astype(int) + \
                   (iny & (b0 <= tx_) & (b1 >= tx_)).astype(int)
            if not mult.any():
                continue
            r = np.repeat(np.arange(m), mult)
            keys.append((ty, tx_))
            rows.append(r)
    return {k: r.astype(np.intp) for k, r in zip(keys, rows)}


def _alphas(pr: Prep, rows, pcx, pcy, dt):
    """(alpha, alpha_raw, g, dx, dy), each (K, P) in dtype dt
    (rasterizer.py:169-184).  Operation order matters for the f32 path."""
    w = pr.w
    mx = pr.mean2d[rows, 0].astype(dt)[:, None]
    my = pr.mean2d[rows, 1].astype(dt)[:, None]
    ca = pr.conic[rows, 0].astype(dt)[:, None]
    cb = pr.conic[rows, 1].astype(dt)[:, None]
    cc = pr.conic[rows, 2].astype(dt)[:, None]
    dx = np.remainder(pcx[None, :] - mx + w / 2.0, w) - w / 2.0
    dy = pcy[None, :] - my
    q = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy
    g = np.exp(-0.5 * q)
    a_raw = pr.opac[rows].astype(dt)[:, None] * g
    a = np.minimum(a_raw, dt(ALPHA_MAX))
    a[a < ALPHA_MIN] = 0.0
    return a, a_raw, g, dx, dy


def _tile_px(ty, tx_, w, h):
    ys = np.arange(ty * TILE, min((ty + 1) * TILE, h))
    xs = np.arange(tx_ * TILE, min((tx_ + 1) * TILE, w))
    return ys, xs


@dataclass
class Aux:
    """Forward state for the backward (rasterizer.py:148-160)."""

    prep: Prep
    tiles: dict
    transmittance: np.ndarray
    contrib_count: np.ndarray
    rx: np.ndarray
    W: np.ndarray
    tx: np.ndarray
    cloud_n: int
    dtype: type
    t_eps: float


def forward(cloud, rx, W, tx, w, h, dtype=np.float32, t_eps=T_EPS,
            threads=1, prep=None):
    """Tiled front-to-back compositing (rasterizer.py:187-234), C channels.
    Returns (img (h,w,C), Aux)."""
    cloud = as_cloud(cloud)
    rx = np.asarray(rx, np.float64).reshape(3)
    W = np.asarray(W, np.float64).reshape(3, 3)
    tx = np.asarray(tx, np.float64).reshape(3)
    pr = prep if prep is not None else prepare(cloud, rx, W, tx, w, h)
    C = cloud.mlp_dims[2]
    img = np.zeros((h, w, C), dtype=dtype)
    T = np.ones((h, w), dtype=dtype)
    cnt = np.zeros((h, w), dtype=np.int32)
    if pr.idx.size == 0:
        return img, Aux(pr, {}, T, cnt, rx, W, tx, cloud.n, dtype, t_eps)
    bins = tile_bins(pr)
    coef = (pr.s / pr.d_tx[:, None]).astype(dtype)

    def run(key):
        ys, xs = _tile_px(key[0], key[1], w, h)
        rows = bins[key]
        gx, gy = np.meshgrid((xs + 0.5).astype(dtype), (ys + 0.5).astype(dtype))
        a = _alphas(pr, rows, gx.ravel(), gy.ravel(), dtype)[0]
        om = 1.0 - a
        tb = np.ones_like(a)
        if a.shape[0] > 1:
            tb[1:] = np.cumprod(om[:-1], axis=0)
        live = tb >= t_eps
        act = live & (a > 0.0)
        wgt = np.where(act, tb * a, dtype(0.0))
        shape = (len(ys), len(xs))
        return (ys, xs, (wgt.T @ coef[rows]).reshape(shape + (C,)),
                np.prod(np.where(live, om, dtype(1.0)), axis=0).reshape(shape),
                act.sum(axis=0, dtype=np.int32).reshape(shape))

    keys = sorted(bins)
    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            outs = list(ex.map(run, keys))
    else:
        outs = [run(k) for k in keys]
    for ys, xs, ti, tf, tc in outs:
        img[np.ix_(ys, xs)] += ti
        T[np.ix_(ys, xs)] = tf
        cnt[np.ix_(ys, xs)] = tc
    return img, Aux(pr, bins, T, cnt, rx, W, tx, cloud.n, dtype, t_eps)


def reference_render(cloud, rx, W, tx, w, h, row_chunk=8):
    """Brute force f64, no tiling, no early exit (rasterizer.py:237-259)."""
    cloud = as_cloud(cloud)
    rx = np.asarray(rx, np.float64).reshape(3)
    W = np.asarray(W, np.float64).reshape(3, 3)
    pr = prepare(cloud, rx, W, tx, w, h)
    C = cloud.mlp_dims[2]
    img = np.zeros((h, w, C))
    if pr.idx.size == 0:
        return img
    coef = pr.s / pr.d_tx[:, None]
    rows = np.arange(pr.idx.size)
    for y0 in range(0, h, row_chunk):
        ys = np.arange(y0, min(y0 + row_chunk, h))
        gx, gy = np.meshgrid(np.arange(w) + 0.5, ys + 0.5)
        a = _alphas(pr, rows, gx.ravel(), gy.ravel(), np.float64)[0]
        tb = np.ones_like(a)
        if a.shape[0] > 1:
            tb[1:] = np.cumprod((1.0 - a)[:-1], axis=0)
        img[ys] = ((tb * a).T @ coef).reshape(len(ys), w, C)
    return img


def zero_grads(cloud: Cloud):
    return {g: np.zeros_like(a, dtype=np.float64)
            for g, a in cloud.groups().items()}


def backward(dL, cloud, tx, aux: Aux):
    """Analytic gradients, f64 recompute per tile + per-Gaussian chain
    (rasterizer.py:262-378).  Returns {group: array}."""
    cloud = as_cloud(cloud)
    tx = np.asarray(tx, np.float64).reshape(3)
    if aux.cloud_n != cloud.n or not np.array_equal(aux.tx, tx):
        raise ValueError("aux does not match this cloud/transmitter")
    grads = zero_grads(cloud)
    pr = aux.prep
    m = pr.idx.size
    if m == 0:
        return grads
    C = cloud.mlp_dims[2]
    dL = np.asarray(dL, np.float64).reshape(pr.h, pr.w, C)
    coef = pr.s / pr.d_tx[:, None]
    g_s = np.zeros((m, C))
    g_sig = np.zeros(m)
    g_con = np.zeros((m, 3))
    g_m2 = np.zeros((m, 2))
    g_d = np.zeros(m)
    for (ty, tx_), rows in sorted(aux.tiles.items()):
        ys, xs = _tile_px(ty, tx_, pr.w, pr.h)
        gx, gy = np.meshgrid(xs + 0.5, ys + 0.5)
        a, a_raw, g, dx, dy = _alphas(pr, rows, gx.ravel().astype(np.float64),
                                      gy.ravel().astype(np.float64), np.float64)
        om = 1.0 - a
        tb = np.ones_like(a)
        if a.shape[0] > 1:
            tb[1:] = np.cumprod(om[:-1], axis=0)
        act = (tb >= aux.t_eps) & (a > 0.0)
        wgt = np.where(act, tb * a, 0.0)
        u = dL[np.ix_(ys, xs)].reshape(-1, C)
        uc = coef[rows] @ u.T
        g_s[rows] += (wgt @ u) / pr.d_tx[rows, None]
        g_d[rows] -= (wgt * (pr.s[rows] @ u.T)).sum(axis=1) / pr.d_tx[rows] ** 2
        tk = wgt * uc
        after = np.flip(np.cumsum(np.flip(tk, 0), axis=0), 0) - tk
        d_a = np.where(act, tb * uc - after / np.maximum(om, 1e-12), 0.0)
        d_sg = np.where(a_raw < ALPHA_MAX, d_a, 0.0)
        g_sig[rows] += (d_sg * g).sum(axis=1)
        d_q = -0.5 * (d_sg * pr.opac[rows][:, None]) * g
        g_con[rows, 0] += (d_q * dx * dx).sum(axis=1)
        g_con[rows, 1] += (d_q * dx * dy).sum(axis=1)
        g_con[rows, 2] += (d_q * dy * dy).sum(axis=1)
        ca = pr.conic[rows, 0][:, None]
        cb = pr.conic[rows, 1][:, None]
        cc = pr.conic[rows, 2][:, None]
        g_m2[rows, 0] -= (d_q * 2.0 * (ca * dx + cb * dy)).sum(axis=1)
        g_m2[rows, 1] -= (d_q * 2.0 * (cb * dx + cc * dy)).sum(axis=1)
    return gaussian_chain(cloud, tx, aux, g_s, g_sig, g_con, g_m2, g_d)


def gaussian_chain(cloud, tx, aux, g_s, g_sig, g_con, g_m2, g_d):
    """Per-Gaussian chain from screen-space grads to parameters
    (rasterizer.py:328-377)."""
    pr = aux.prep
    W = aux.W
    m = pr.idx.size
    A = np.empty((m, 2, 2))
    A[:, 0, 0], A[:, 0, 1], A[:, 1, 0], A[:, 1, 1] = (
        pr.conic[:, 0], pr.conic[:, 1], pr.conic[:, 1], pr.conic[:, 2])
    GA = np.empty((m, 2, 2))
    GA[:, 0, 0], GA[:, 0, 1], GA[:, 1, 0], GA[:, 1, 1] = (
        g_con[:, 0], g_con[:, 1], g_con[:, 1], g_con[:, 2])
    G2 = -np.einsum("mij,mjk,mkl->mil", A, GA, A)
    J = pr.J
    S3 = covariance3d(cloud)[pr.idx]
    M3 = np.einsum("ij,mjk,lk->mil", W, S3, W)
    GM3 = np.einsum("mai,mab,mbl->mil", J, G2, J)
    GJ = 2.0 * np.einsum("mab,mbj,mjk->mak", G2, J, M3)
    g_mu = np.einsum("mkj,mkji->mi", GJ, jacobian_hessian(pr.mu_v, pr.w, pr.h))
    GS = np.einsum("ji,mjk,kl->mil", W, GM3, W)
    R = quat_to_rot(unit_quat(cloud.rotations[pr.idx]))
    sc = np.exp(cloud.log_scales[pr.idx])
    GM = 2.0 * np.einsum("mij,mjk->mik", GS, R * sc[:, None, :])
    g_ls = np.einsum("mik,mik->mk", R, GM) * sc
    g_q = quat_grad(cloud.rotations[pr.idx], GM * sc[:, None, :])
    g_w, g_in = mlp_bwd(cloud.mlp_weights[pr.idx], pr.inputs, g_s,
                        cloud.mlp_dims)
    g_mu += view_angles_grad(pr.mu_v, g_in[:, 3], g_in[:, 4])
    g_mu += np.einsum("mki,mk->mi", J, g_m2)
    g_pos = g_mu @ W
    diff = cloud.positions[pr.idx] - aux.tx
    g_pos += np.where(~pr.d_clamped, g_d, 0.0)[:, None] * diff / \
        pr.d_tx[:, None]
    g_raw = g_sig * pr.opac * (1.0 - pr.opac)
    out = zero_grads(cloud)
    np.add.at(out["positions"], pr.idx, g_pos)
    np.add.at(out["log_scales"], pr.idx, g_ls)
    np.add.at(out["rotations"], pr.idx, g_q)
    np.add.at(out["raw_opacities"], (pr.idx, 0), g_raw)
    np.add.at(out["mlp_weights"], pr.idx, g_w)
    return out


def check_finite(grads):
    """rasterizer.py:63-66."""
    for k in GROUPS:
        if not np.all(np.isfinite(grads[k])):
            raise FloatingPointError(f"non-finite gradient in {k}")


# ---------------------------------------------------------- image / loss
def magnitude(img):
    """|z| of a 2-channel image (image.py:46-51)."""
    d = np.asarray(img, np.float64)
    if d.shape[-1] != 2:
        raise ValueError("magnitude needs 2 channels")
    return np.hypot(d[..., 0], d[..., 1])[..., None]


def magnitude_grad(img, g):
    """image.py:54-61."""
    d = np.asarray(img, np.float64)
    mag = np.hypot(d[..., 0], d[..., 1])
    g = np.asarray(g, np.float64).reshape(mag.shape)
    k = np.where(mag > 0.0, g / np.where(mag > 0.0, mag, 1.0), 0.0)
    return np.stack([d[..., 0] * k, d[..., 1] * k], axis=-1)


def _win():
    x = np.arange(SSIM_WIN) - (SSIM_WIN - 1) / 2.0
    k = np.exp(-0.5 * (x / SSIM_SIG) ** 2)
    return k / k.sum()


_WIN = _win()
_HALF = (SSIM_WIN - 1) // 2


def blur(x):
    """Separable window, scipy 'reflect' padding (optimize.py:91-94)."""
    from scipy.ndimage import correlate1d
    return correlate1d(correlate1d(x, _WIN, axis=0, mode="reflect"), _WIN,
                       axis=1, mode="reflect")


def blur_adjoint(g):
    """Adjoint of blur (optimize.py:97-115)."""
    from scipy.ndimage import correlate1d
    for ax in (0, 1):
        pad = [(0, 0)] * g.ndim
        pad[ax] = (_HALF, _HALF)
        z = correlate1d(np.pad(g, pad), _WIN, axis=ax, mode="constant")
        z = np.moveaxis(z, ax, 0)
        n = z.shape[0] - 2 * _HALF
        f = z[_HALF:_HALF + n].copy()
        f[:_HALF] += z[:_HALF][::-1]
        f[n - _HALF:] += z[_HALF + n:][::-1]
        g = np.moveaxis(f, 0, ax)
    return g


def ssim_and_grad(x, y):
    """(mean SSIM, d/dx) for one channel (optimize.py:118-162)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    c1, c2 = SSIM_K1 ** 2, SSIM_K2 ** 2
    mx, my = blur(x), blur(y)
    vx = blur(x * x) - mx * mx
    vy = blur(y * y) - my * my
    vxy = blur(x * y) - mx * my
    a1, a2 = 2 * mx * my + c1, 2 * vxy + c2
    b1, b2 = mx * mx + my * my + c1, vx + vy + c2
    s = (a1 * a2) / (b1 * b2)
    da1, da2 = a2 / (b1 * b2), a1 / (b1 * b2)
    db1, db2 = -s / b1, -s / b2
    g_mx = 2 * my * da1 - 2 * my * da2 + 2 * mx * db1 - 2 * mx * db2
    gr = (blur_adjoint(g_mx) + 2 * x * blur_adjoint(db2)
          + y * blur_adjoint(2 * da2)) / s.size
    return float(s.mean()), gr


def ssim(x, y):
    """Mean SSIM, per-channel average for 3-D input (optimize.py:134-142)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if x.ndim == 3:
        return float(np.mean([ssim(x[:, :, c], y[:, :, c])
                              for c in range(x.shape[2])]))
    return ssim_and_grad(x, y)[0]


def loss_and_grad(pred, gt, lam):
    """(1-lam) L1 + lam (1-SSIM) and d/dpred (optimize.py:165-188)."""
    p = np.asarray(pred, np.float64)
    g = np.asarray(gt, np.float64)
    if p.shape != g.shape:
        raise ValueError("image shape mismatch")
    two_d = p.ndim == 2
    if two_d:
        p, g = p[:, :, None], g[:, :, None]
    diff = p - g
    l1 = float(np.mean(np.abs(diff)))
    grad = (1.0 - lam) * np.sign(diff) / diff.size
    vals = []
    for ch in range(p.shape[2]):
        v, gr = ssim_and_grad(p[:, :, ch], g[:, :, ch])
        vals.append(v)
        grad[:, :, ch] -= lam * gr / p.shape[2]
    loss = (1.0 - lam) * l1 + lam * (1.0 - float(np.mean(vals)))
    return loss, (grad[:, :, 0] if two_d else grad)


def psnr(pred, gt):
    m = float(np.mean((np.asarray(pred, np.float64) -
                       np.asarray(gt, np.float64)) ** 2))
    return math.inf if m == 0.0 else 10.0 * math.log10(1.0 / m)


# ---------------------------------------------------------------- Adam
@dataclass
class AdamCfg:
    """Subset of TrainConfig used by the update (optimize.py:27-49)."""

    position_lr_init: float = 0.0016
    position_lr_final: float = 1.6e-6
    position_lr_delay_mult: float = 0.01
    position_lr_max_steps: int = 30000
    opacity_lr: float = 0.0055
    scaling_lr: float = 0.005
    rotation_lr: float = 0.001
    mlp_lr: float = 0.002
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-15


def position_lr(step, cfg):
    """optimize.py:205-213."""
    t = float(np.clip(step / cfg.position_lr_max_steps, 0.0, 1.0))
    lr = math.exp((1.0 - t) * math.log(cfg.position_lr_init)
                  + t * math.log(cfg.position_lr_final))
    ramp = float(np.clip(step / (0.01 * cfg.position_lr_max_steps), 0.0, 1.0))
    return (cfg.position_lr_delay_mult + (1.0 - cfg.position_lr_delay_mult)
            * math.sin(0.5 * math.pi * ramp)) * lr


def group_lr(name, step, cfg):
    """optimize.py:216-222."""
    return {"positions": None, "log_scales": cfg.scaling_lr,
            "rotations": cfg.rotation_lr, "raw_opacities": cfg.opacity_lr,
            "mlp_weights": cfg.mlp_lr}[name] if name != "positions" \
        else position_lr(step, cfg)


def adam_update(cloud: Cloud, grads, m, v, step, cfg):
    """In-place Adam with per-group LR + quaternion renorm
    (optimize.py:234-259)."""
    check_finite(grads)
    b1, b2, eps = cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
    t = step + 1
    for name, p in cloud.groups().items():
        lr = group_lr(name, step, cfg)
        g = grads[name]
        m[name] *= b1
        m[name] += (1 - b1) * g
        v[name] *= b2
        v[name] += (1 - b2) * g * g
        p -= lr * (m[name] / (1 - b1 ** t)) / \
            (np.sqrt(v[name] / (1 - b2 ** t)) + eps)
    cloud.rotations[:] = unit_quat(cloud.rotations)


# ------------------------------------------------------ scene generation
def make_uniform(lo, hi, n, seed, init_scale=None, logit=-2.0,
                 mlp_dims=DEFAULT_MLP_DIMS):
    """Seeded uniform cloud, PCG64 stream (scene.py:184-207)."""
    lo = np.asarray(lo, np.float64).reshape(3)
    hi = np.asarray(hi, np.float64).reshape(3)
    if init_scale is None:
        init_scale = 0.02 * float(np.linalg.norm(hi - lo))
    rng = np.random.Generator(np.random.PCG64(seed))
    pos = rng.uniform(lo, hi, size=(n, 3))
    ls = np.full((n, 3), np.log(init_scale))
    rot = np.zeros((n, 4))
    rot[:, 0] = 1.0
    op = np.full((n, 1), float(logit))
    mw = rng.standard_normal((n, n_mlp_params(mlp_dims)))
    return Cloud(pos, ls, rot, op, mw, tuple(mlp_dims))


def round_f32(cloud: Cloud):
    """GSPC round trip: every parameter f32-representable
    (scene.py:210-239)."""
    return Cloud(*(getattr(cloud, g).astype(np.float32).astype(np.float64)
                   for g in GROUPS), mlp_dims=cloud.mlp_dims)


def bench_scene(n, F=1, seed=0):
    """Reference bench scene (cli.py:239-246) with mlp_out = 2F, GSPC-rounded
    (SURVEY.md 8(d))."""
    c = make_uniform([-5, -0.2, -5], [5, 3.2, 5], n, seed,
                     mlp_dims=(5, 16, 2 * F))
    c.mlp_weights *= 0.3
    return round_f32(c)


def perturbed_scene(n, seed, spread=4.0, scale=0.3, mlp_scale=0.3,
                    min_height=0.3, max_height=3.0, F=1):
    """tests/conftest.py:15-27 recipe."""
    rng = np.random.default_rng(seed)
    c = make_uniform([-spread, min_height, -spread],
                     [spread, max_height, spread], n, seed, init_scale=scale,
                     mlp_dims=(5, 16, 2 * F))
    c.mlp_weights *= mlp_scale
    c.raw_opacities[:] = rng.normal(0.0, 1.0, (n, 1))
    c.rotations += rng.normal(0.0, 0.3, (n, 4))
    c.log_scales += rng.normal(0.0, 0.4, (n, 3))
    return c


def sample_tx(seed, n, lo=(-4.0, 0.0, -4.0), hi=(4.0, 2.0, 4.0),
              rx=(0.0, 0.0, 0.0), keepout=1.0):
    """Rejection-sampled TX positions (rfsim.py:120-128)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rx = np.asarray(rx, np.float64)
    out = np.empty((n, 3))
    i = 0
    while i < n:
        p = rng.uniform(lo, hi)
        if np.linalg.norm(p - rx) >= keepout:
            out[i] = p
            i += 1
    return out


def pixel_dir(u, v, w, h):
    """geometry.py:83-95 (used to build known-answer scenes)."""
    az = ((np.asarray(u, np.float64) + 0.5) * 2.0 / w - 1.0) * np.pi
    el = (np.asarray(v, np.float64) + 0.5) * (np.pi / 2.0) / h
    ce = np.cos(el)
    return np.stack([ce * np.sin(az), np.sin(el), ce * np.cos(az)], axis=-1)


def write_gspc(path, cloud: Cloud):
    """GSPC v1 writer (scene.py:210-218)."""
    i, h, o = cloud.mlp_dims
    with open(path, "wb") as f:
        f.write(b"GSPC" + struct.pack("<5I", 1, cloud.n, i, h, o))
        for g in GROUPS:
            f.write(np.ascontiguousarray(getattr(cloud, g), "<f4").tobytes())


def live_fraction(aux: Aux):
    """Share of kept Gaussians with at least one included contribution
    (SURVEY.md 8(d)); recomputed from the tile lists."""
    pr = aux.prep
    m = pr.idx.size
    if m == 0:
        return 0.0
    live = np.zeros(m, bool)
    w, h = pr.w, pr.h
    for (ty, tx_), rows in aux.tiles.items():
        ys, xs = _tile_px(ty, tx_, w, h)
        gx, gy = np.meshgrid((xs + 0.5).astype(aux.dtype),
                             (ys + 0.5).astype(aux.dtype))
        a = _alphas(pr, rows, gx.ravel(), gy.ravel(), aux.dtype)[0]
        tb = np.ones_like(a)
        if a.shape[0] > 1:
            tb[1:] = np.cumprod((1.0 - a)[:-1], axis=0)
        act = (tb >= aux.t_eps) & (a > 0.0)
        live[rows[act.any(axis=1)]] = True
    return float(live.mean())


def cpu_threads():
    return os.cpu_count() or 1


# ------------------------------------------------- rfsim / RFSI wire format
RSSI_FLOOR_DB = -100.0


def free_space_amp(d, wavelength):
    """rfsim.py:65-71."""
    d = np.asarray(d, np.float64)
    return (wavelength / (4.0 * np.pi * d)) * np.exp(-2j * np.pi * d / wavelength)


def ground_truth(emitters, rx, wavelength, tx, w, h, scale=None):
    """Closed-form multipath magnitude (rfsim.py:75-99).  emitters: list of
    (position[3], complex gain, angular spread).  Returns (h, w) f64."""
    tx = np.asarray(tx, np.float64).reshape(3)
    rx = np.asarray(rx, np.float64).reshape(3)
    uu, vv = np.meshgrid(np.arange(w), np.arange(h))
    dirs = pixel_dir(uu.ravel(), vv.ravel(), w, h)
    field = np.zeros(w * h, dtype=np.complex128)
    for pos, gain, spread in emitters:
        pos = np.asarray(pos, np.float64)
        to_em = pos - rx
        r_em = np.linalg.norm(to_em)
        if r_em < 1e-9:
            continue
        path = np.linalg.norm(pos - tx) + r_em
        amp = gain * free_space_amp(path, wavelength)
        cosang = np.clip(dirs @ (to_em / r_em), -1.0, 1.0)
        ang = np.arccos(cosang)
        field += amp * np.exp(-ang * ang / (2.0 * spread ** 2))
    mag = np.abs(field).reshape(h, w)
    return mag / scale if scale is not None else mag


def select_pixels(seed, w, h, fraction):
    """The PCG64 pixel subset of rssi_from_spectrum (rfsim.py:215-218,230)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_total = w * h
    return rng.choice(n_total, size=int(np.ceil(fraction * n_total)),
                      replace=False)


def energy_db(energy, offset=0.0):
    """rfsim.py:221-224."""
    return RSSI_FLOOR_DB if energy <= 0.0 else 10.0 * np.log10(energy) + offset


def rssi(img, fraction, seed, offset=0.0):
    """rssi_from_spectrum (rfsim.py:227-243); img (h, w, c), c = 1 or 2."""
    d = np.asarray(img, np.float64)
    e = d[:, :, 0] ** 2 + d[:, :, 1] ** 2 if d.shape[2] == 2 else d[:, :, 0] ** 2
    sel = select_pixels(seed, d.shape[1], d.shape[0], fraction)
    return energy_db(float(e.reshape(-1)[sel].sum()) / fraction, offset)


def write_rfsi(path, data):
    """RFSI v1 writer (image.py:64-69)."""
    d = np.asarray(data)
    h, w, c = d.shape
    with open(path, "wb") as f:
        f.write(b"RFSI" + struct.pack("<4I", 1, w, h, c))
        f.write(np.ascontiguousarray(d, "<f4").tobytes())


def read_rfsi(path):
    """RFSI v1 reader (image.py:72-86)."""
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:4] == b"RFSI"
    ver, w, h, c = struct.unpack("<4I", buf[4:20])
    assert ver == 1
    return np.frombuffer(buf, "<f4", count=w * h * c, offset=20).reshape(h, w, c)
