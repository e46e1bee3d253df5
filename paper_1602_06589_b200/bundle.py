"""System bundles and the build flow of the reference CLI on the B200 path.

A bundle (reference `cli.py:203-280`) is a directory with ``manifest.json``,
``layout.json`` (block heights, capacity height, ‖u̇‖ per row, l_sph, l_nonsph),
``A.hsm1`` / ``B.hsm1`` (the stacked coefficients, R x N_G), per-atom
``T_AA_xxx.hsm1`` / ``T_AB_xxx.hsm1`` / ``T_BB_xxx.hsm1`` and, for physics bundles,
``system.json``.

`build_bundle` is `hsdla build` (`cmd_build`, `cli.py:310-328`): the stacks go from
disk straight into HBM, the fused native build runs, and H and S stream from HBM into
``H.hsm1`` / ``S.hsm1`` next to ``report.json`` — no host copy of any N_G x N_G
matrix.  `load_bundle` / `write_bundle` are the host-side readers and writers
(`cli.py:248-280`, `:203-245`).
"""
from __future__ import annotations

import hashlib
import json
import time
from pathlib import Path

import numpy as np

from . import device
from .builder import (BuildConfig, BuildReport, StackedCoefficients, TMatrixSet, _t_sizes,
                      estimate_memory, fill_report)
from .errors import ConfigurationError, ContractViolationError
from .flapw import SystemSpec
from .hsm1 import read_hsm1, read_hsm1_device, write_hsm1, write_hsm1_device
from .kernels import get_backend
from .matrix import AtomBlockLayout, ComplexDense

BUNDLE_FORMAT = "hsdla-bundle-v1"


def _sha256(path: Path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for block in iter(lambda: fh.read(1 << 24), b""):
            h.update(block)
    return "sha256:" + h.hexdigest()


def _read_layout(bundle_dir: Path):
    manifest_path = bundle_dir / "manifest.json"
    if not manifest_path.is_file():
        raise OSError(f"{bundle_dir} has no manifest.json")
    json.loads(manifest_path.read_text())  # malformed manifest -> JSONDecodeError
    doc = json.loads((bundle_dir / "layout.json").read_text())
    layout = AtomBlockLayout(tuple(doc["block_heights"]), int(doc["capacity_block_height"]))
    return layout, doc


def _read_tmats(bundle_dir: Path, layout: AtomBlockLayout, doc: dict) -> TMatrixSet:
    t_aa, t_ab, t_bb = [], [], []
    for a in range(layout.atom_count):
        t_aa.append(read_hsm1(bundle_dir / f"T_AA_{a:03d}.hsm1"))
        t_ab.append(read_hsm1(bundle_dir / f"T_AB_{a:03d}.hsm1"))
        t_bb.append(read_hsm1(bundle_dir / f"T_BB_{a:03d}.hsm1"))
    return TMatrixSet(t_aa=t_aa, t_ab=t_ab, t_bb=t_bb, l_sph=list(doc["l_sph"]),
                      l_nonsph=list(doc["l_nonsph"]))


def _read_spec(bundle_dir: Path):
    path = bundle_dir / "system.json"
    return SystemSpec.from_json(path.read_text()) if path.is_file() else None


def load_bundle(bundle_dir):
    """(spec or None, StackedCoefficients, TMatrixSet) on the host (`cli.py:248-280`);
    A*/B* are re-embedded into capacity-height allocations as the reference does."""
    bundle_dir = Path(bundle_dir)
    layout, doc = _read_layout(bundle_dir)
    a_c = read_hsm1(bundle_dir / "A.hsm1")
    b_c = read_hsm1(bundle_dir / "B.hsm1")
    a_star = ComplexDense.zeros(a_c.rows, a_c.cols, capacity_rows=layout.capacity_rows)
    b_star = ComplexDense.zeros(b_c.rows, b_c.cols, capacity_rows=layout.capacity_rows)
    a_star.array[:] = a_c.array
    b_star.array[:] = b_c.array
    coeffs = StackedCoefficients(a_star, b_star, layout, np.asarray(doc["udot_norms"]))
    return _read_spec(bundle_dir), coeffs, _read_tmats(bundle_dir, layout, doc)


def write_bundle(outdir, coeffs: StackedCoefficients, tmats: TMatrixSet, spec=None, *,
                 seed: int = 0, params: dict | None = None) -> dict:
    """Write a bundle readable by the reference CLI and by `build_bundle` (`cli.py:203-245`);
    returns the manifest."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    files = {}

    def emit_matrix(name, m):
        write_hsm1(outdir / name, m)
        files[name] = _sha256(outdir / name)

    def emit_text(name, text):
        (outdir / name).write_text(text)
        files[name] = _sha256(outdir / name)

    if spec is not None:
        emit_text("system.json", spec.to_json())
    layout_doc = {
        "block_heights": list(coeffs.layout.block_heights),
        "capacity_block_height": coeffs.layout.capacity_block_height,
        "udot_norms": np.asarray(coeffs.udot_norms).tolist(),
        "l_sph": list(tmats.l_sph),
        "l_nonsph": list(tmats.l_nonsph),
    }
    emit_text("layout.json", json.dumps(layout_doc, sort_keys=True))
    emit_matrix("A.hsm1", coeffs.A_star)
    emit_matrix("B.hsm1", coeffs.B_star)
    for a in range(tmats.atom_count):
        emit_matrix(f"T_AA_{a:03d}.hsm1", tmats.t_aa[a])
        emit_matrix(f"T_AB_{a:03d}.hsm1", tmats.t_ab[a])
        emit_matrix(f"T_BB_{a:03d}.hsm1", tmats.t_bb[a])
    manifest = {"format": BUNDLE_FORMAT, "seed": seed, "params": dict(params or {}),
                "n_basis": coeffs.n_basis, "files": files}
    (outdir / "manifest.json").write_text(json.dumps(manifest, sort_keys=True, indent=1))
    return manifest


def _regenerator(spec):
    """The A*/B* re-creation callback of the backup=False flow (`cli.py:283-292`): refills the
    caller's stacks from the bundle's system.json by compute_AB; None without a spec."""
    if spec is None:
        return None

    def regen(coeffs):
        from .flapw import compute_AB

        fresh = compute_AB(spec)
        coeffs.A_star.array[:] = fresh.A_star.array
        coeffs.B_star.array[:] = fresh.B_star.array

    return regen


def _run_dir(out, seed: int) -> Path:
    if out:
        path = Path(out)
    else:
        path = Path("hsdla-runs") / f"{time.strftime('%Y%m%d-%H%M%S')}-seed{seed}"
    path.mkdir(parents=True, exist_ok=True)
    return path


def build_bundle(bundle_dir, out=None, *, backup: bool = True, threads: int = 1,
                 backend: str = "optimized", seed: int = 0) -> tuple[Path, BuildReport]:
    """`hsdla build BUNDLE` on the GPU: writes H.hsm1, S.hsm1, report.json; returns
    (output directory, report).

    Same configuration errors as `cmd_build` (`cli.py:310-318`): backup=False needs a
    bundle with system.json.  The device build never consumes its inputs, so both backup
    modes produce bitwise identical files (as the reference's do)."""
    from .pipeline import build_device, pack_tmats, padded_ld

    bundle_dir = Path(bundle_dir)
    layout, doc = _read_layout(bundle_dir)
    spec = _read_spec(bundle_dir)
    if not backup and spec is None:
        raise ConfigurationError(
            "backup=false needs a bundle with system.json to re-create coefficients")
    config = BuildConfig(backup=backup, thread_count=threads, backend=backend)
    be = get_backend(config.backend, config.thread_count)
    tmats = _read_tmats(bundle_dir, layout, doc)
    outdir = _run_dir(out, seed)

    t = device.require_cuda()
    t0 = time.perf_counter()
    r = layout.total_rows
    ld = padded_ld(r)
    a_d, ra, n = read_hsm1_device(bundle_dir / "A.hsm1", ld)
    b_d, rb, nb = read_hsm1_device(bundle_dir / "B.hsm1", ld)
    udot_host = np.asarray(doc["udot_norms"], dtype=np.float64)
    # StackedCoefficients' shape contract (builder.py:54-65), checked on the device stacks
    if ra != r or rb != r:
        raise ContractViolationError(
            f"stacked matrices must expose {r} rows, got {ra} and {rb}")
    if nb != n:
        raise ContractViolationError("A_star and B_star need equal column counts")
    if udot_host.shape != (r,):
        raise ContractViolationError(
            f"udot_norms must have one entry per row ({r}), got {udot_host.shape}")
    sizes = _t_sizes(_ShapeOnly(layout, n), tmats)
    udot = t.zeros(ld, dtype=t.float64, device="cuda")
    udot[:r] = t.from_numpy(np.ascontiguousarray(udot_host)).to("cuda")
    h_d = device.empty_matrix(n, n, n)
    s_d = device.empty_matrix(n, n, n)
    res, ws = build_device(n_basis=n, heights=layout.block_heights,
                           row_offset=layout.offsets[:-1], tpack=pack_tmats(tmats), A=a_d, B=b_d,
                           Bs=None, udot=udot, ld=ld, force_general_path=False, H=h_d, S=s_d,
                           ldh=n)
    write_hsm1_device(outdir / "H.hsm1", h_d, n, n)
    write_hsm1_device(outdir / "S.hsm1", s_d, n, n)
    wall = time.perf_counter() - t0
    report = BuildReport(thread_count=be.threads)
    report.predicted_bytes = estimate_memory(layout.atom_count, layout.capacity_block_height, n,
                                             backup)
    fill_report(report, res, layout, sizes, n, config, wall,
                int(sum(x.numel() * x.element_size() for x in (a_d, b_d, udot, h_d, s_d))
                    + ws.numel()))
    (outdir / "report.json").write_text(json.dumps(report.to_json_dict(), sort_keys=True,
                                                   indent=1))
    return outdir, report


class _ShapeOnly:
    """The two attributes `_t_sizes` reads from StackedCoefficients."""

    def __init__(self, layout, n):
        self.layout = layout
        self.n_basis = n
