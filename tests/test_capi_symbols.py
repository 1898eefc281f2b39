"""CPU: the in-tree C-ABI library loads and exports every symbol include/*.h declares."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(gpmppi_[a-z0-9_]+)\s*\(", src):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2411_03289_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) > 40
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _capi.SIGNATURES}
    assert syms <= bound, sorted(syms - bound)


def test_library_loads_and_fails_loudly_without_gpu():
    import numpy as np
    import pytest
    import paper_2411_03289_b200 as G
    assert G._capi.lib().gpmppi_abi_version() == 2
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(G.CudaError):
        G.GpModel.fit(np.zeros((1, 4)), np.ones((1, 1)), [G.KernelParams()])


def test_host_tuple_combine_matches_direct_softmax():
    """Sharded reduction algebra on CPU: combining per-shard tuples
    equals the single-shard weights/update (mppi.cpp:125-164)."""
    import numpy as np
    import paper_2411_03289_b200 as G
    rng = np.random.default_rng(0)
    K, T, lam = 300, 7, 0.1
    c = rng.uniform(0, 5, K)
    c[[3, 77]] = np.nan
    eps = rng.standard_normal((K, T, 2))

    def tup(cs, es):
        f = np.isfinite(cs)
        m = cs[f].min() if f.any() else np.inf
        e = np.where(f, np.exp(-(np.where(f, cs, m) - m) / lam), 0.0)
        S = (e[:, None, None] * es).sum(0).ravel()
        return np.concatenate([[m, e.sum(), (e * e).sum(), (e * np.where(f, cs - m, 0)).sum(),
                                f.sum(), np.where(f, cs, 0).sum()], S])
    full = tup(c, eps)
    parts = np.stack([tup(c[a:b], eps[a:b]) for a, b in ((0, 100), (100, 250), (250, 300))])
    comb = G.combine_tuples(parts, T, lam)
    np.testing.assert_allclose(comb, full, rtol=1e-12, atol=1e-12)
    w = np.where(np.isfinite(c), np.exp(-(np.nan_to_num(c, nan=np.inf) - np.nanmin(c)) / lam), 0)
    w /= w.sum()
    np.testing.assert_allclose(comb[6:].reshape(T, 2), (w[:, None, None] * eps).sum(0) * comb[1],
                               rtol=1e-10)
