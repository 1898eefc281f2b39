"""Regenerates tests/golden/ref_rng.npz from the reference's own RNG header.

Run in the build container (needs /root/reference): it compiles
/root/reference/proj/include/gpmppi/rng.hpp via oracle/build_ref.sh into
oracle/_ref/libref_rng.so and records derive_seed values, raw uniform and
Gaussian streams, and K×T×2 perturbation tensors (mppi.cpp:53-62 layout
[s][k][channel]) for a few (seed, tick) pairs. The committed .npz is what the
tests compare the oracle (and the device noise-injection path) against.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    subprocess.run([os.path.join(ROOT, "oracle", "build_ref.sh")], check=True)
    so = os.path.join(ROOT, "oracle", "_ref", "libref_rng.so")
    if not os.path.exists(so):
        sys.exit("reference RNG not buildable here")
    L = C.CDLL(so)
    dp = C.POINTER(C.c_double)
    L.ref_derive_seed.restype = C.c_uint64
    L.ref_derive_seed.argtypes = [C.c_uint64] * 3
    L.ref_uniform_stream.argtypes = [C.c_uint64, C.c_int, dp]
    L.ref_gaussian_stream.argtypes = [C.c_uint64, C.c_int, dp]
    L.ref_sample_perturbations.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                           C.c_uint64, dp]
    triples = np.array([[0, 0, 0], [1, 2, 3], [12345, 7, 100], [2**63 + 5, 2**40, 17],
                        [11, 0, 4095]], dtype=np.uint64)
    derived = np.array([L.ref_derive_seed(int(a), int(b), int(c)) for a, b, c in triples],
                       dtype=np.uint64)
    uni = np.empty((3, 700))
    gau = np.empty((3, 701))
    for i, seed in enumerate((0, 5489, 2**64 - 1)):
        L.ref_uniform_stream(seed, 700, uni[i].ctypes.data_as(dp))
        L.ref_gaussian_stream(seed, 701, gau[i].ctypes.data_as(dp))
    cases = [(64, 8, 0.09, 0.25, 12345, 3), (257, 6, 0.09, 0.25, 12345, 0),
             (100, 40, 0.04, 0.16, 11, 9)]
    eps = {}
    for j, (K, T, sv2, sw2, seed, tick) in enumerate(cases):
        e = np.empty((K, T, 2))
        L.ref_sample_perturbations(K, T, sv2, sw2, seed, tick, e.ctypes.data_as(dp))
        eps[f"eps{j}"] = e
    np.savez_compressed(os.path.join(HERE, "ref_rng.npz"), triples=triples, derived=derived,
                        uniform=uni, gaussian=gau, cases=np.array(cases, dtype=np.float64),
                        **eps)
    print("wrote", os.path.join(HERE, "ref_rng.npz"))


if __name__ == "__main__":
    main()
