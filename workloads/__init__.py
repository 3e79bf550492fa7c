"""Seeded synthetic workloads for the SFSeg power-iteration hot path.

This module is shared by the tests, ``bench.py`` and the CPU oracle's callers.
It holds NO arithmetic of the method (no Gaussian taps, no combine, no power
iteration, no threshold): only configuration presets and seeded input
generators, so that the oracle (``oracle/``) and the CUDA path
(``paper_2212_08058_b200``) can be fed identical fp32 bits without sharing code.

The paper's data (DAVIS-2016 soft masks from 15 methods, tracker crops) is not
available; these generators stand in for it (DESIGN.md
"Input recipe"):

* c1 tiny     -- BASELINE.json configs[0]: 1x8x32x32, C=1, U[0,1] smoothed by an
                 in-bounds 3x3 box mean, seed 0.
* c2 video    -- configs[1]: 1x70x480x854, C=1, 1-3 ellipse blobs moving
                 ~3 px/frame (value 0.9), background U[0,0.2], noise N(0,0.05^2),
                 clipped to [0,1].  Stands in for a DAVIS-2016 video (480x854,
                 ~69 frames) with one method's soft mask.
* c3 ensemble -- configs[2]: c2 blobs, C=6 perturbed copies (offset +-10 px,
                 noise 0.1, 10 % dropped frames); w = softmax(N(0, I_6)).
                 Stands in for the 15-method SFSeg++ ensemble.
* c4 tracking -- configs[3]: 64 volumes 32x256x256, C=4, one blob random-walking
                 2 px/frame.  Stands in for SFTrack++ crops.
* c5 long     -- configs[4]: 1x512x1080x1920, C=2, c2 generator at 1080p.
* probe       -- c2 data with the paper's own 3x7x7 support.

Randomness (SURVEY.md §8(d) generator rules): numpy ``Generator(PCG64)``;
global parameters from ``default_rng([seed, cfg])``; per-frame values from
``default_rng([seed, cfg, 1 + c, t])`` so any frame can be produced
independently (time-slab ranks generate only their slab plus halo).
All values are computed in float64 and cast once to float32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = ["Config", "CONFIGS", "get_config", "generate", "Workload"]


@dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int               # integer used in the RNG keys
    B: int
    T: int
    H: int
    W: int
    C: int
    sigma_t: float
    sigma_s: float
    radius_t: int             # ceil(3 sigma_t)
    radius_s: int             # ceil(3 sigma_s)
    K: int                    # power iterations
    tau: float = 0.5          # threshold (A12: per-frame max rescale)
    act: int = 0              # 0 identity, 1 sigmoid  (A2: configs use identity, b = 0)
    bias: float = 0.0
    backward: bool = False    # config asks for dL/dw (c3)
    note: str = ""

    @property
    def N(self) -> int:
        return self.B * self.T * self.H * self.W

    @property
    def voxels_per_volume(self) -> int:
        return self.T * self.H * self.W


CONFIGS = {
    "c1": Config("c1", 1, 1, 8, 32, 32, 1, 1.0, 2.0, 3, 6, 10,
                 note="BASELINE configs[0]: tiny volume, dense 8192x8192 check"),
    "c2": Config("c2", 2, 1, 70, 480, 854, 1, 2.0, 8.0, 6, 24, 15,
                 note="BASELINE configs[1]: video-segmentation volume"),
    "c3": Config("c3", 3, 1, 70, 480, 854, 6, 2.0, 8.0, 6, 24, 15, backward=True,
                 note="BASELINE configs[2]: SFSeg++ ensemble, forward + dL/dw"),
    "c4": Config("c4", 4, 64, 32, 256, 256, 4, 1.5, 6.0, 5, 18, 10,
                 note="BASELINE configs[3]: 64 tracking crops"),
    "c5": Config("c5", 5, 1, 512, 1080, 1920, 2, 3.0, 12.0, 9, 36, 20,
                 note="BASELINE configs[4]: long 1080p volume"),
    "probe": Config("probe", 2, 1, 70, 480, 854, 1, 0.5, 1.0, 1, 3, 15,
                    note="supplementary: c2 data with the paper's 3x7x7 support (PAPER.md:319)"),
    # the full SFSeg operator; S = the c2 soft mask, F = two
    # optical-flow-magnitude stand-ins (direct / reverse), p = 0.2,
    # alpha = 1, N_i = 5 iterations
    "c2f": Config("c2f", 6, 1, 70, 480, 854, 1, 2.0, 8.0, 6, 24, 5,
                  note="f1: full SFSeg operator on the c2 volume (S = soft mask, F = 2 flow-magnitude maps)"),
}

# full-operator hyper-parameters of "c2f" (alpha = 1, p = 0.2 semi-supervised)
FULL_P = 0.2
FULL_ALPHA = 1.0


def get_config(name: str, **overrides) -> Config:
    base = CONFIGS[name]
    if not overrides:
        return base
    d = dict(base.__dict__)
    d.update(overrides)
    return Config(**d)


# ----------------------------------------------------------------------------
# blob geometry (pure data synthesis: ellipses at integer pixel centres)
# ----------------------------------------------------------------------------

def _reflect(p: float, lo: float, hi: float) -> float:
    """Reflect a linearly moving coordinate into [lo, hi] (triangle wave)."""
    L = hi - lo
    if L <= 0:
        return lo
    q = (p - lo) % (2.0 * L)
    if q > L:
        q = 2.0 * L - q
    return lo + q


@dataclass
class _Blob:
    cy: float
    cx: float
    a: float          # semi-axis along the rotated x direction
    b: float          # semi-axis along the rotated y direction
    theta: float
    vy: float = 0.0
    vx: float = 0.0
    path: Optional[np.ndarray] = None   # explicit [T][2] centres (random walk)

    def centre(self, t: int, H: int, W: int):
        if self.path is not None:
            return float(self.path[t, 0]), float(self.path[t, 1])
        return (_reflect(self.cy + self.vy * t, 0.0, H - 1.0),
                _reflect(self.cx + self.vx * t, 0.0, W - 1.0))


def _paint(mask: np.ndarray, blob: _Blob, cy: float, cx: float) -> None:
    """OR an ellipse into ``mask`` (membership tested at integer pixel centres)."""
    H, W = mask.shape
    ext = max(blob.a, blob.b) + 1.0
    y0, y1 = max(0, int(math.floor(cy - ext))), min(H, int(math.ceil(cy + ext)) + 1)
    x0, x1 = max(0, int(math.floor(cx - ext))), min(W, int(math.ceil(cx + ext)) + 1)
    if y0 >= y1 or x0 >= x1:
        return
    yy = np.arange(y0, y1, dtype=np.float64)[:, None] - cy
    xx = np.arange(x0, x1, dtype=np.float64)[None, :] - cx
    c, s = math.cos(blob.theta), math.sin(blob.theta)
    u = (xx * c + yy * s) / blob.a
    v = (-xx * s + yy * c) / blob.b
    mask[y0:y1, x0:x1] |= (u * u + v * v) <= 1.0


def _blob_mask(blobs: Sequence[_Blob], t: int, H: int, W: int,
               offset=(0, 0)) -> np.ndarray:
    m = np.zeros((H, W), dtype=bool)
    for bl in blobs:
        cy, cx = bl.centre(t, H, W)
        _paint(m, bl, cy + offset[0], cx + offset[1])
    return m


def _video_blobs(seed: int, cfg_id: int, H: int, W: int, axes, speed) -> list:
    rng = np.random.default_rng([seed, cfg_id])
    n = int(rng.integers(1, 4))
    blobs = []
    for _ in range(n):
        a, b = rng.uniform(axes[0], axes[1], size=2)
        theta = rng.uniform(0.0, math.pi)
        cy = rng.uniform(0.2 * H, 0.8 * H)
        cx = rng.uniform(0.2 * W, 0.8 * W)
        direction = rng.uniform(0.0, 2.0 * math.pi)
        sp = rng.uniform(speed[0], speed[1])
        blobs.append(_Blob(cy, cx, a, b, theta, sp * math.sin(direction), sp * math.cos(direction)))
    return blobs


def _soft_frame(mask: np.ndarray, rng: np.random.Generator, noise: float) -> np.ndarray:
    """0.9 inside the blob union, U[0,0.2] background, + N(0, noise^2), clip [0,1]."""
    H, W = mask.shape
    bg = rng.random((H, W)) * 0.2
    base = np.where(mask, 0.9, bg)
    return np.clip(base + rng.normal(0.0, noise, size=(H, W)), 0.0, 1.0)


# ----------------------------------------------------------------------------
# public generator
# ----------------------------------------------------------------------------

@dataclass
class Workload:
    cfg: Config
    ch: np.ndarray                  # float32 [B][C][T][H][W] (T = the generated range)
    w: np.ndarray                   # float32 [C]
    b: float
    mask: Optional[np.ndarray]      # bool [B][T][H][W] clean blob union (c2/c3/c4/c5)
    t0: int = 0                     # first generated frame
    extra: dict = field(default_factory=dict)


def _c1(seed: int) -> np.ndarray:
    raw = np.random.default_rng(seed).random((8, 32, 32))
    out = np.empty_like(raw)
    T, H, W = raw.shape
    # per-frame 3x3 box mean over in-bounds neighbours only (count varies at borders)
    for y in range(H):
        for x in range(W):
            ys, ye = max(0, y - 1), min(H, y + 2)
            xs, xe = max(0, x - 1), min(W, x + 2)
            out[:, y, x] = raw[:, ys:ye, xs:xe].reshape(T, -1).mean(axis=1)
    return out


def generate(name: str, seed: int = 0, t_range: Optional[tuple] = None,
             volumes: Optional[Sequence[int]] = None, cfg: Optional[Config] = None,
             with_mask: bool = True) -> Workload:
    """Generate the fp32 channel stack of config ``name``.

    ``t_range=(t0, t1)`` generates only frames [t0, t1) (frame-addressable; used
    for time-slab crops and halos).  ``volumes`` selects volume indices for c4.
    ``cfg`` may override shape fields (e.g. a cropped H/W for quick tests) while
    keeping the recipe of ``name``.
    """
    cfg = cfg or CONFIGS[name]
    T, H, W, C = cfg.T, cfg.H, cfg.W, cfg.C
    t0, t1 = (0, T) if t_range is None else t_range
    assert 0 <= t0 <= t1 <= T
    nt = t1 - t0
    recipe = name if name in ("c1", "c2", "c3", "c4", "c5") else "c2"
    if name == "c2f":
        # unary map S: the c2 soft mask; pairwise channels F: flow-magnitude stand-ins --
        # 0.5 (~3 px/frame of a 6 px/frame scale) where the blob union of frames t and
        # t+1 (direct) / t-1 and t (reverse) moves, background U[0,0.05] + N(0,0.02^2), clip
        base = generate("c2", seed, t_range, cfg=get_config("c2", T=T, H=H, W=W), with_mask=with_mask)
        blobs = _video_blobs(seed, 2, H, W, (24.0, 72.0), (2.5, 3.5))
        f_ch = np.empty((1, 2, nt, H, W), np.float32)
        for i, t in enumerate(range(t0, t1)):
            m0 = _blob_mask(blobs, t, H, W)
            for c, t2 in enumerate((t + 1, t - 1)):
                moving = m0 | _blob_mask(blobs, t2, H, W)
                rng = np.random.default_rng([seed, 6, 1 + c, t])
                bg = rng.random((H, W)) * 0.05
                f_ch[0, c, i] = np.clip(np.where(moving, 0.5, bg) + rng.normal(0.0, 0.02, (H, W)), 0.0, 1.0)
        return Workload(cfg, base.ch, base.w, 0.0, base.mask, t0,
                        {"f_ch": f_ch, "wf": np.array([0.5, 0.5], np.float32), "p": FULL_P, "alpha": FULL_ALPHA})

    if recipe == "c1":
        if (T, H, W, C) != (8, 32, 32, 1):
            raise ValueError("c1 recipe is fixed at 1x8x32x32, C=1")
        vol = _c1(seed)[t0:t1]
        ch = vol[None, None].astype(np.float32)
        return Workload(cfg, ch, np.ones(1, np.float32), 0.0, None, t0)

    if recipe in ("c2", "c3"):
        blobs = _video_blobs(seed, 2, H, W, (24.0, 72.0), (2.5, 3.5))
        ch = np.empty((1, C, nt, H, W), np.float32)
        mask = np.empty((1, nt, H, W), bool) if with_mask else None
        if recipe == "c2":
            offsets = [(0, 0)]
            w = np.ones(1, np.float32)
        else:
            grng = np.random.default_rng([seed, 3])
            offsets = [tuple(int(v) for v in grng.integers(-10, 11, size=2)) for _ in range(C)]
            z = np.random.default_rng([seed, 3, 99]).normal(size=C)
            e = np.exp(z - z.max())
            w = (e / e.sum()).astype(np.float32)
        for i, t in enumerate(range(t0, t1)):
            clean = _blob_mask(blobs, t, H, W)
            if mask is not None:
                mask[0, i] = clean
            for c in range(C):
                rng = np.random.default_rng([seed, cfg.cfg_id if recipe == "c3" else 2, 1 + c, t])
                if recipe == "c2":
                    ch[0, c, i] = _soft_frame(clean, rng, 0.05)
                else:
                    drop = rng.random() < 0.1
                    m = _blob_mask(blobs, t, H, W, offsets[c])
                    f = _soft_frame(m, rng, 0.1)
                    ch[0, c, i] = 0.0 if drop else f
        return Workload(cfg, ch, w, cfg.bias, mask, t0, {"offsets": offsets})

    if recipe == "c4":
        vols = list(range(cfg.B)) if volumes is None else list(volumes)
        ch = np.empty((len(vols), C, nt, H, W), np.float32)
        mask = np.empty((len(vols), nt, H, W), bool) if with_mask else None
        for j, v in enumerate(vols):
            rng = np.random.default_rng([seed, 4, v])
            a, b = rng.uniform(20.0, 40.0, size=2)
            theta = rng.uniform(0.0, math.pi)
            ang = rng.uniform(0.0, 2.0 * math.pi, size=max(T - 1, 0))
            path = np.empty((T, 2))
            path[0] = (H / 2.0, W / 2.0)
            for t in range(1, T):
                path[t, 0] = _reflect(path[t - 1, 0] + 2.0 * math.sin(ang[t - 1]), 0.0, H - 1.0)
                path[t, 1] = _reflect(path[t - 1, 1] + 2.0 * math.cos(ang[t - 1]), 0.0, W - 1.0)
            blob = _Blob(0.0, 0.0, a, b, theta, path=path)
            for i, t in enumerate(range(t0, t1)):
                clean = _blob_mask([blob], t, H, W)
                if mask is not None:
                    mask[j, i] = clean
                for c in range(C):
                    frng = np.random.default_rng([seed, 4, v, 1 + c, t])
                    ch[j, c, i] = _soft_frame(clean, frng, 0.05)
        w = np.full(C, 1.0 / C, np.float32)
        return Workload(cfg, ch, w, cfg.bias, mask, t0, {"volumes": vols})

    # c5: c2 generator scaled x2.25 at 1080p; ch1 is a c3-style perturbed copy
    blobs = _video_blobs(seed, 5, H, W, (54.0, 162.0), (5.0, 7.0))
    off = tuple(int(v) for v in np.random.default_rng([seed, 5, 99]).integers(-10, 11, size=2))
    ch = np.empty((1, C, nt, H, W), np.float32)
    mask = np.empty((1, nt, H, W), bool) if with_mask else None
    for i, t in enumerate(range(t0, t1)):
        clean = _blob_mask(blobs, t, H, W)
        if mask is not None:
            mask[0, i] = clean
        ch[0, 0, i] = _soft_frame(clean, np.random.default_rng([seed, 5, 1, t]), 0.05)
        if C > 1:
            rng = np.random.default_rng([seed, 5, 2, t])
            drop = rng.random() < 0.1
            f = _soft_frame(_blob_mask(blobs, t, H, W, off), rng, 0.1)
            ch[0, 1, i] = 0.0 if drop else f
    w = np.full(C, 1.0 / C, np.float32)
    return Workload(cfg, ch, w, cfg.bias, mask, t0, {"offset": off})


def random_volume(shape, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Plain U[lo,hi) fp32 array for small property / edge-case tests."""
    return (np.random.default_rng(seed).random(shape) * (hi - lo) + lo).astype(np.float32)
