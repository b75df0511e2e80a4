"""Shared helpers for the parity tests: run the GPU path (C-ABI), the oracle
restatement in GPU reduction order, and the reference, on the same inputs."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk
from paper_1905_01549_b200.cgvk import Precond, Variant, Vec

ALL_VARIANTS = list(Variant)
VEC_IDS = list(Vec)


def tree_dot(A_dev: cgvk.DeviceMatrix):
    block, gmax, order = A_dev.reduction_config()
    return ("tree", block, gmax, order)


def gpu_state(s: cgvk.Solver) -> dict:
    st, sc, stats = s._status()
    return {"k": st.k, "state": st.state, "breakdown": st.breakdown, "criterion": st.criterion,
            "allocated_vectors": st.allocated_vectors,
            "scalars": {f: getattr(sc, f) for f in O.SCALAR_NAMES},
            "stats": {f: getattr(stats, f) for f in ("spmv_calls", "block_spmv_calls",
                                                      "precond_applies", "reductions")}}


def gpu_vectors(s: cgvk.Solver) -> dict:
    out = {}
    for w in VEC_IDS:
        try:
            out[int(w)] = s.vector(w)
        except cgvk.InvalidArgument:
            out[int(w)] = None
    return out


def oracle_vectors(o) -> dict:
    return {w: o.vector(w) for w in range(11)}


def same_bits(a, b) -> bool:
    if a is None or b is None:
        return a is None and b is None
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def compare_states(g: dict, o: dict, where: str) -> None:
    for key in ("k", "state", "breakdown", "criterion", "allocated_vectors", "stats"):
        assert g[key] == o[key], f"{where}: {key} gpu={g[key]} oracle={o[key]}"
    for name, ov in o["scalars"].items():
        gv = g["scalars"][name]
        assert same_bits(np.float64(gv), np.float64(ov)) or (np.isnan(gv) and np.isnan(ov)), \
            f"{where}: scalar {name} gpu={gv!r} oracle={ov!r}"


def compare_vectors(g: dict, o: dict, where: str) -> None:
    for w in range(11):
        assert same_bits(g[w], o[w]), f"{where}: vector {O.VEC_NAMES[w]} differs"


def lockstep(A, A_dev, variant, precond, b, x0, steps, cfg_kwargs=None, check_vectors_every=1):
    """Step the GPU solver and the tree-order restatement side by side and
    demand bit-identical state after initialize and after every step."""
    cfg_kwargs = cfg_kwargs or {}
    cfg = cgvk.VariantConfig.make(variant)
    for k_, v_ in cfg_kwargs.items():
        setattr(cfg, k_, v_)
    s = cgvk.initialize(cfg, A_dev, precond, b, x0)
    o = O.Restatement(A, int(variant), int(precond), b, x0, dot=tree_dot(A_dev),
                      nu_expr=int(cfg.nu_expression), recompute_nu=cfg.recompute_nu,
                      recompute_w=cfg.recompute_w, unsimplified_mu=cfg.unsimplified_mu,
                      track_delta=cfg.track_delta)
    tag = f"{variant.name}/{Precond(precond).name}"
    compare_states(gpu_state(s), o.state(), f"{tag} init")
    compare_vectors(gpu_vectors(s), oracle_vectors(o), f"{tag} init")
    for k in range(1, steps + 1):
        if o.state()["state"] != 0:
            break
        cgvk.step(s)
        o.step()
        compare_states(gpu_state(s), o.state(), f"{tag} k={k}")
        if k % check_vectors_every == 0 or o.state()["state"] != 0:
            compare_vectors(gpu_vectors(s), oracle_vectors(o), f"{tag} k={k}")
    return s, o
