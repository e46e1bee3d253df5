"""Shared test configuration.

`-m "not gpu"` runs here without a GPU: oracle vs golden fixtures, host logic, C-ABI
symbol checks, multi-rank (gloo) sharding logic.  `-m gpu` tests are the parity tests
proper: they call the sm_100a library through its C ABI and compare with the oracle
(`oracle/`, test infrastructure) and the golden fixtures made by the real reference.
"""
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhsdla_b200.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def rand_complex(rng, rows, cols):
    return rng.standard_normal((rows, cols)) + 1j * rng.standard_normal((rows, cols))


def rel_fro(x, y):
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), np.finfo(float).tiny))


def hermitian_from_lower(t):
    full = np.tril(t) + np.tril(t, -1).conj().T
    np.fill_diagonal(full, full.diagonal().real)
    return full


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def spec_from_golden(d, prefix="spec_"):
    """Rebuild the product SystemSpec stored by tests/golden/make_golden.py."""
    from paper_1602_06589_b200 import RadialBoundaryData, SystemSpec

    l_sph = d[prefix + "l_sph"]
    radial = []
    for a, l in enumerate(l_sph):
        n = int(l) + 1
        kw = {f: d[f"{prefix}rad_{f}"][a, :n] for f in ("u", "u_prime", "udot", "udot_prime",
                                                        "udot_norm")}
        radial.append(RadialBoundaryData(energy=np.zeros(n), **kw))
    return SystemSpec(positions=d[prefix + "positions"], rotations=d[prefix + "rotations"],
                      mt_radius=d[prefix + "mt_radius"], l_sph=l_sph, l_nonsph=l_sph,
                      k_point=np.zeros(3), k_vectors=d[prefix + "k_vectors"],
                      omega=float(d[prefix + "omega"]), radial=radial)


def build_case(d, ci):
    """(heights, cap, force, A, B, udot, t_aa, t_ab, t_bb, H, S, ledger, mask) of build_small case ci."""
    p = f"c{ci}_"
    heights = [int(h) for h in d[p + "heights"]]
    fam = {f: [d[f"{p}{f}_{a}"] for a in range(len(heights))] for f in ("t_aa", "t_ab", "t_bb")}
    return dict(heights=heights, cap=int(d[p + "cap"]), force=bool(d[p + "force"]),
                A=d[p + "A"], B=d[p + "B"], udot=d[p + "udot"], t_aa=fam["t_aa"],
                t_ab=fam["t_ab"], t_bb=fam["t_bb"], H=d[p + "H"], S=d[p + "S"],
                ledger=d[p + "ledger"], mask=[bool(x) for x in d[p + "hpd_mask"]])


LEDGER_KEYS = ("hermitian_rank_k", "hermitian_rank_2k", "general_product", "hermitian_product",
               "triangular_product", "cholesky", "row_scale")
