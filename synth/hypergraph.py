"""Synthetic image-tagging hypergraphs shaped like the paper's workloads.

The paper's dataset (a private Flickr "Greek places" crawl, PAPER.md:183-208,
Table 1) is not available; these seeded inputs stand in for it, with the
shapes BASELINE.json `configs[0..4]` name (recipe: DESIGN.md "Input recipe",
SURVEY.md §8(d)).  Vertices are images; hyperedges are

  * visual: one per vertex, {v} U kNN_K(v) over Gaussian-mixture features,
  * tags:   Zipf(s) popularity, P(v has t) = min(1, 3 p_t)  (mean 3 tags/vertex),
  * groups: G user groups, size ~ U{8..40}, members uniform without replacement,

H(v, e) = 1 iff v in e.  Column order [visual | tags | groups].
The RHS Y is the N x T tag matrix (0/1), T = number of tag hyperedges.

No step of the method is computed here (no degrees, no Theta, no Omega).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class SynthConfig:
    name: str
    N: int          # vertices (images)
    d: int          # feature dimension
    C: int          # feature clusters
    K: int          # visual kNN
    n_tag: int      # tag hyperedges (= T)
    zipf_s: float   # tag popularity exponent
    G: int          # user groups
    unit_w: bool    # unit hyperedge weights (else U(0.5, 1.5))
    b: int          # diagonal block size
    k: int          # rank
    q: int          # subspace-iteration passes (Alg. 1 loop bound)
    mu: float = 1.0  # the regulariser theta ("mu=1", configs[0]); c = mu/(1+mu)
    seed: int = 0

    @property
    def T(self) -> int:
        return self.n_tag

    @property
    def nb(self) -> int:
        return self.N // self.b

    def with_(self, **kw) -> "SynthConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; unstated values inherit from the nearest earlier
# config.
CONFIGS: Dict[int, SynthConfig] = {
    1: SynthConfig("cfg1", N=512, d=64, C=8, K=5, n_tag=20, zipf_s=1.1, G=16,
                   unit_w=True, b=128, k=32, q=2),
    2: SynthConfig("cfg2", N=4096, d=128, C=32, K=10, n_tag=100, zipf_s=1.1, G=200,
                   unit_w=False, b=256, k=64, q=2),
    3: SynthConfig("cfg3", N=16384, d=256, C=64, K=10, n_tag=500, zipf_s=1.0, G=1000,
                   unit_w=False, b=512, k=128, q=3),
    4: SynthConfig("cfg4", N=65536, d=256, C=128, K=15, n_tag=1000, zipf_s=1.0, G=4000,
                   unit_w=False, b=1024, k=256, q=3),
    5: SynthConfig("cfg5", N=32768, d=256, C=128, K=15, n_tag=1000, zipf_s=1.0, G=4000,
                   unit_w=False, b=1024, k=256, q=2),
}


def cfg5_points() -> List[Tuple[int, int, int]]:
    """The 36 (b, k, q) sweep points of configs[4] (all have k <= b)."""
    return [(b, k, q) for b in (512, 1024, 2048) for k in (64, 128, 256, 512)
            for q in (1, 2, 4) if k <= b]


@dataclasses.dataclass
class HypergraphInput:
    cfg: SynthConfig
    row_ptr: np.ndarray   # int64 [N+1]  CSR over vertices
    col_idx: np.ndarray   # int32 [nnz]  hyperedge ids, strictly increasing per row
    w: np.ndarray         # float32 [E]  hyperedge weights
    Y: np.ndarray         # float32 [N, T] tag-label right-hand sides (0/1)

    @property
    def N(self) -> int:
        return self.row_ptr.shape[0] - 1

    @property
    def E(self) -> int:
        return self.w.shape[0]

    @property
    def nnz(self) -> int:
        return self.col_idx.shape[0]


def _knn(x: np.ndarray, K: int) -> np.ndarray:
    """Indices [N, K] of the K nearest neighbours (Euclidean, self excluded)."""
    N = x.shape[0]
    try:
        import torch
        dev = "cuda" if torch.cuda.is_available() and N > 4096 else "cpu"
        xt = torch.from_numpy(x).to(dev)
        if dev == "cpu" and N <= 4096:
            xt = xt.double()
        sq = (xt * xt).sum(1)
        out = torch.empty((N, K), dtype=torch.int64)
        chunk = 2048
        for i0 in range(0, N, chunk):
            i1 = min(N, i0 + chunk)
            d2 = sq[i0:i1, None] + sq[None, :] - 2.0 * (xt[i0:i1] @ xt.T)
            d2[torch.arange(i1 - i0, device=dev), torch.arange(i0, i1, device=dev)] = float("inf")
            idx = torch.topk(d2, K, dim=1, largest=False, sorted=True).indices
            out[i0:i1] = idx.cpu()
        return out.numpy()
    except ImportError:  # pragma: no cover - torch is always present in this image
        sq = (x.astype(np.float64) ** 2).sum(1)
        out = np.empty((N, K), dtype=np.int64)
        for i0 in range(0, N, 512):
            i1 = min(N, i0 + 512)
            d2 = sq[i0:i1, None] + sq[None, :] - 2.0 * (x[i0:i1].astype(np.float64) @ x.T.astype(np.float64))
            d2[np.arange(i1 - i0), np.arange(i0, i1)] = np.inf
            out[i0:i1] = np.argsort(d2, axis=1, kind="stable")[:, :K]
        return out


def make_input(cfg: SynthConfig) -> HypergraphInput:
    """Draw (H, w, Y) for `cfg` from numpy PCG64(cfg.seed); deterministic."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    N, d = cfg.N, cfg.d
    # Gaussian-mixture features: x_v = mu_{c(v)} + 0.5 * N(0, I_d)
    cl = rng.integers(0, cfg.C, size=N)
    centres = rng.standard_normal((cfg.C, d)).astype(np.float32)
    feats = centres[cl] + 0.5 * rng.standard_normal((N, d)).astype(np.float32)
    feats = np.ascontiguousarray(feats, dtype=np.float32)
    nn = _knn(feats, cfg.K)                                   # [N, K]
    # tag matrix: p_t ~ t^-s (normalised), P(v has t) = min(1, 3 p_t)
    t = np.arange(1, cfg.n_tag + 1, dtype=np.float64)
    p = t ** (-cfg.zipf_s)
    p /= p.sum()
    prob = np.minimum(1.0, 3.0 * p)
    tags = rng.random((N, cfg.n_tag)) < prob[None, :]
    empty = np.nonzero(~tags.any(axis=0))[0]
    for tcol in empty:                                         # an empty tag gets one random vertex
        tags[rng.integers(0, N), tcol] = True
    # user groups
    sizes = rng.integers(8, 41, size=cfg.G)
    groups = [rng.choice(N, size=int(s), replace=False) for s in sizes]
    E = N + cfg.n_tag + cfg.G
    if cfg.unit_w:
        w = np.ones(E, dtype=np.float32)
    else:
        w = rng.uniform(0.5, 1.5, size=E).astype(np.float32)

    # COO incidence (vertex, edge)
    vis_v = np.concatenate([np.arange(N, dtype=np.int64), nn.reshape(-1)])
    vis_e = np.concatenate([np.arange(N, dtype=np.int64), np.repeat(np.arange(N, dtype=np.int64), cfg.K)])
    tv, tt = np.nonzero(tags)
    tag_v = tv.astype(np.int64)
    tag_e = N + tt.astype(np.int64)
    grp_v = np.concatenate(groups).astype(np.int64) if groups else np.zeros(0, np.int64)
    grp_e = N + cfg.n_tag + np.repeat(np.arange(cfg.G, dtype=np.int64), sizes)
    V = np.concatenate([vis_v, tag_v, grp_v])
    Ecol = np.concatenate([vis_e, tag_e, grp_e])
    key = np.unique(V * E + Ecol)                              # sorted, deduplicated
    rows = key // E
    cols = (key % E).astype(np.int32)
    row_ptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=N), out=row_ptr[1:])
    Y = np.ascontiguousarray(tags, dtype=np.float32)
    return HypergraphInput(cfg, row_ptr, cols, w, Y)


def make_tiny(N: int, b: int, k: int, q: int, *, K: int = 3, n_tag: int = 8, G: int = 3,
              d: int = 8, C: int = 2, unit_w: bool = False, seed: int = 0) -> HypergraphInput:
    """A small hypergraph with the same recipe (tests; group sizes capped at N)."""
    cfg = SynthConfig(f"tiny{N}", N=N, d=d, C=C, K=K, n_tag=n_tag, zipf_s=1.1, G=G,
                      unit_w=unit_w, b=b, k=k, q=q, seed=seed)
    if N < 41:
        # groups draw sizes in 8..40 without replacement: keep them feasible
        cfg = cfg.with_(G=0)
    return make_input(cfg)
