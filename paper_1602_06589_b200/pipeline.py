"""Device-resident H/S setup pipeline (the B200 hot path).

    SystemSpec + T blocks --(H2D, tiny)--> [A/B generator] --> [native build] --> H, S in HBM

`HSPipeline` owns the HBM buffers for one problem shape and runs one k-point per
call: the fused A/B generator (reference `flapw.py:201-233`) writes A, B and the
row-scaled B directly, then `hsdla_build_hs` (reference `builder.py:403-474`) runs
the T-block applications and the two triangular DMMA contractions with the
Hermitian mirror fused into their epilogue.  Inputs stay resident; nothing but the
spec, the T blocks and (optionally) the results crosses PCIe.

Layout in HBM (column-major complex128, leading dimension `ld` = R rounded up to a
multiple of 16 so every 16-element K chunk starts on a 256-byte boundary):
A, B, B_scaled, Z, XY: ld x N_G each; H, S: N_G x N_G (ld = N_G); T forms:
n_tsets x 4 x m_max^2.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native, device
from .errors import ContractViolationError, NativeLibraryError

LD_ALIGN = 16


def padded_ld(rows: int) -> int:
    return max(LD_ALIGN, (rows + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN)


@dataclass
class TPack:
    """Distinct T sets uploaded once: atoms sharing the same T objects share a set."""

    t_index: np.ndarray  # (n_atoms,) int32
    t_dim: np.ndarray    # (n_tsets,) int32
    t_ld: int
    t_aa: object         # device tensors (n_tsets, t_ld, t_ld) complex128, column-major per set
    t_ab: object
    t_bb: object
    h2d_bytes: int

    @property
    def n_tsets(self) -> int:
        return int(self.t_dim.shape[0])


def pack_tmats(tmats) -> TPack:
    """Deduplicate per-atom T blocks by identity and upload them (one H2D per family)."""
    t = device.require_cuda()
    keys, index, reps = {}, [], []
    for a in range(tmats.atom_count):
        key = (id(tmats.t_aa[a]), id(tmats.t_ab[a]), id(tmats.t_bb[a]))
        if key not in keys:
            keys[key] = len(reps)
            reps.append(a)
        index.append(keys[key])
    dims = np.array([tmats.t_aa[a].rows for a in reps], dtype=np.int32)
    t_ld = int(max(1, dims.max()))
    host = np.zeros((3, len(reps), t_ld, t_ld), dtype=np.complex128)
    for s, a in enumerate(reps):
        m = int(dims[s])
        for f, fam in enumerate((tmats.t_aa, tmats.t_ab, tmats.t_bb)):
            host[f, s, :m, :m] = fam[a].array.T  # (col, row) storage = column-major
    dev = t.from_numpy(host).to("cuda")
    return TPack(np.array(index, dtype=np.int32), dims, t_ld, dev[0], dev[1], dev[2],
                 host.nbytes)


def build_device(*, n_basis, heights, row_offset, tpack: TPack, A, B, Bs, udot, ld,
                 force_general_path, H, S, ldh, shard_rank=0, n_shards=1, workspace=None,
                 ab_args=None, host_out=None):
    """Run `hsdla_build_hs` (or `hsdla_setup_hs` when `ab_args` is given: A/B generation
    fused in front) on device buffers; returns (result dict, workspace tensor)."""
    lib = _native.load()
    t = device.require_cuda()
    na = len(heights)
    h_arr = np.ascontiguousarray(heights, dtype=np.int32)
    o_arr = np.ascontiguousarray(row_offset, dtype=np.int64)
    ti = np.ascontiguousarray(tpack.t_index, dtype=np.int32)
    td = np.ascontiguousarray(tpack.t_dim, dtype=np.int32)
    args = _native.BuildArgs()
    args.n_atoms = na
    args.n_basis = n_basis
    args.heights = h_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.row_offset = o_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    args.t_index = ti.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.n_tsets = tpack.n_tsets
    args.t_dim = td.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.t_aa = tpack.t_aa.data_ptr()
    args.t_ab = tpack.t_ab.data_ptr()
    args.t_bb = tpack.t_bb.data_ptr()
    args.t_ld = tpack.t_ld
    args.A = A.data_ptr()
    args.B = B.data_ptr()
    args.B_scaled = Bs.data_ptr() if Bs is not None else None
    args.udot_norms = udot.data_ptr() if udot is not None else None
    args.ld = ld
    args.force_general_path = 1 if force_general_path else 0
    args.H = H.data_ptr()
    args.S = S.data_ptr()
    args.ldh = ldh
    args.shard_rank = shard_rank
    args.n_shards = n_shards
    if host_out is not None:  # pinned (n, n) tensors: D2H overlapped inside the native call
        args.H_host = host_out[0].data_ptr()
        args.S_host = host_out[1].data_ptr()
        args.ldh_host = int(host_out[0].shape[1])
    need = lib.hsdla_build_workspace_size(ctypes.byref(args))
    if workspace is None or workspace.numel() < need:
        workspace = t.empty(max(need, 1), dtype=t.uint8, device="cuda")
    args.workspace = workspace.data_ptr()
    args.workspace_bytes = workspace.numel()
    mask = (ctypes.c_int32 * na)()
    info = (ctypes.c_int32 * tpack.n_tsets)()
    res = _native.BuildResult()
    res.hpd_mask = mask
    res.chol_info = info
    if ab_args is not None:
        rc = lib.hsdla_setup_hs(device.ctx(), ctypes.byref(ab_args), ctypes.byref(args),
                                ctypes.byref(res))
    else:
        rc = lib.hsdla_build_hs(device.ctx(), ctypes.byref(args), ctypes.byref(res))
    if rc == _native.HSDLA_ERR_NAN_INPUT:
        raise ContractViolationError("NaN in Cholesky input (lower triangle)")
    if rc == _native.HSDLA_ERR_NONFINITE:
        raise ContractViolationError("accumulator contains non-finite values")
    _native.check(rc, "hsdla_build_hs")
    out = {
        "hpd_mask": [bool(mask[i]) for i in range(na)],
        "chol_info": [int(info[i]) for i in range(tpack.n_tsets)],
        "ms": {"setup": res.ms_setup, "S": res.ms_S, "H_ABBA_BB": res.ms_H_ABBA_BB,
               "H_AA": res.ms_H_AA},
        "kernel_ms": {"contract_S": res.ms_contract_S, "contract_H": res.ms_contract_H,
                      "apply_Z": res.ms_apply_Z, "apply_XY": res.ms_apply_XY},
        "workspace_bytes": int(need),
        "ms_total": res.ms_total,
    }
    return out, workspace


class DeviceSpec:
    """A SystemSpec's arrays in HBM (k-vectors, positions, rotations, radii, radial table)."""

    def __init__(self, spec):
        t = device.require_cuda()
        self.n_atoms = int(spec.n_atoms)
        self.n_basis = int(spec.n_basis)
        self.l_sph = np.ascontiguousarray(spec.l_sph, dtype=np.int32)
        if self.l_sph.max() > _native.MAX_LSPH:
            raise NativeLibraryError(f"l_sph > {_native.MAX_LSPH} is not compiled in")
        heights = (self.l_sph.astype(np.int64) + 1) ** 2
        self.heights = heights.astype(np.int32)
        self.row_offset = np.concatenate(([0], np.cumsum(heights)[:-1])).astype(np.int64)
        self.rows = int(heights.sum())
        stride = int(self.l_sph.max()) + 1
        radial = np.zeros((self.n_atoms, stride, 5))
        for a, rad in enumerate(spec.radial):
            n = int(self.l_sph[a]) + 1
            radial[a, :n, 0] = rad.u[:n]
            radial[a, :n, 1] = rad.u_prime[:n]
            radial[a, :n, 2] = rad.udot[:n]
            radial[a, :n, 3] = rad.udot_prime[:n]
            radial[a, :n, 4] = rad.udot_norm[:n]
        self.radial_stride = stride
        host = [np.ascontiguousarray(spec.k_vectors, dtype=np.float64),
                np.ascontiguousarray(spec.positions, dtype=np.float64),
                np.ascontiguousarray(np.asarray(spec.rotations, dtype=np.float64).reshape(-1, 9)),
                np.ascontiguousarray(spec.mt_radius, dtype=np.float64),
                radial]
        self.h2d_bytes = int(sum(h.nbytes for h in host))
        self.kv, self.pos, self.rot, self.rmt, self.radial = (
            t.from_numpy(h).to("cuda", non_blocking=False) for h in host)
        self.omega = float(spec.omega)


def make_ab_args(dspec: DeviceSpec, A, B, Bs, ld, udot) -> "_native.AbArgs":
    """C argument block of the A/B generator (host arrays stay alive on `dspec`)."""
    args = _native.AbArgs()
    args.n_atoms = dspec.n_atoms
    args.n_basis = dspec.n_basis
    args.k_vectors = dspec.kv.data_ptr()
    args.positions = dspec.pos.data_ptr()
    args.rotations = dspec.rot.data_ptr()
    args.mt_radius = dspec.rmt.data_ptr()
    args.radial = dspec.radial.data_ptr()
    args.radial_stride = dspec.radial_stride
    l_arr = dspec.l_sph
    o_arr = dspec.row_offset
    args.l_sph = l_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.row_offset = o_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    args.omega = dspec.omega
    args.A = A.data_ptr()
    args.B = B.data_ptr()
    args.B_scaled = Bs.data_ptr() if Bs is not None else None
    args.ld = ld
    args.udot_norms = udot.data_ptr() if udot is not None else None
    return args


def ab_generate_device(dspec: DeviceSpec, A, B, Bs, ld, udot):
    """Fused A/B (+ scaled B, + row norms) generation into device buffers."""
    lib = _native.load()
    args = make_ab_args(dspec, A, B, Bs, ld, udot)
    _native.check(lib.hsdla_ab_generate(device.ctx(), ctypes.byref(args)), "hsdla_ab_generate")


class HSPipeline:
    """Reusable HBM buffers for up to `n_capacity` basis functions and one atom layout;
    `run` = one k-point (any N_G <= n_capacity, e.g. a k-point batch with varying G-sets)."""

    def __init__(self, n_capacity: int, heights, *, shard_rank: int = 0, n_shards: int = 1):
        t = device.require_cuda()
        self.n_capacity = int(n_capacity)
        self.heights = np.asarray(heights, dtype=np.int32)
        self.rows = int(self.heights.sum())
        self.ld = padded_ld(self.rows)
        n = self.n_capacity
        self.A = device.empty_matrix(self.ld, n, self.ld, zero=True)
        self.B = device.empty_matrix(self.ld, n, self.ld, zero=True)
        self.Bs = device.empty_matrix(self.ld, n, self.ld, zero=True)
        self.udot = t.zeros(self.ld, dtype=t.float64, device="cuda")
        self.H = device.empty_matrix(n, n, n)
        self.S = device.empty_matrix(n, n, n)
        self.workspace = None
        self.shard_rank, self.n_shards = shard_rank, n_shards
        self.n_basis = 0

    @property
    def device_bytes(self) -> int:
        tot = sum(x.numel() * x.element_size() for x in (self.A, self.B, self.Bs, self.udot,
                                                          self.H, self.S))
        if self.workspace is not None:
            tot += self.workspace.numel()
        return int(tot)

    def generate(self, dspec: DeviceSpec):
        if dspec.n_basis > self.n_capacity or dspec.rows != self.rows:
            raise ContractViolationError("spec shape does not fit the pipeline buffers")
        self.n_basis = dspec.n_basis
        ab_generate_device(dspec, self.A, self.B, self.Bs, self.ld, self.udot)

    def build(self, dspec: DeviceSpec, tpack: TPack, force_general_path: bool = False):
        res, self.workspace = build_device(
            n_basis=dspec.n_basis, heights=dspec.heights, row_offset=dspec.row_offset, tpack=tpack,
            A=self.A, B=self.B, Bs=self.Bs, udot=self.udot, ld=self.ld,
            force_general_path=force_general_path, H=self.H, S=self.S, ldh=self.n_capacity,
            shard_rank=self.shard_rank, n_shards=self.n_shards, workspace=self.workspace)
        return res

    def run(self, dspec: DeviceSpec, tpack: TPack, force_general_path: bool = False,
            host_out=None):
        """One k-point, spec -> H, S in HBM, as a single native call (`hsdla_setup_hs`).
        With `host_out` = pinned (n, n) tensors, H and S are also copied to the host with the
        copies overlapped with the remaining compute."""
        if dspec.n_basis > self.n_capacity or dspec.rows != self.rows:
            raise ContractViolationError("spec shape does not fit the pipeline buffers")
        self.n_basis = dspec.n_basis
        ab = make_ab_args(dspec, self.A, self.B, self.Bs, self.ld, None)
        res, self.workspace = build_device(
            n_basis=dspec.n_basis, heights=dspec.heights, row_offset=dspec.row_offset, tpack=tpack,
            A=self.A, B=self.B, Bs=self.Bs, udot=self.udot, ld=self.ld,
            force_general_path=force_general_path, H=self.H, S=self.S, ldh=self.n_capacity,
            shard_rank=self.shard_rank, n_shards=self.n_shards, workspace=self.workspace,
            ab_args=ab, host_out=host_out)
        return res

    def launches_per_run(self, dspec: DeviceSpec) -> int:
        """Kernels this pipeline launches per k-point (A/B + row-norm kernel per l group,
        T prep, S contraction, Z apply, XY apply, H contraction)."""
        return len(np.unique(dspec.l_sph)) + 5

    def result_views(self):
        """Host-indexable (n, n) views: H[i, j] == tensor[j, i] (column-major storage)."""
        n = self.n_basis
        return self.H[:n, :n], self.S[:n, :n]


def build_hs(spec, tmats, config=None, *, pipeline: HSPipeline | None = None, host_out=None):
    """spec + T blocks -> (H, S, result) with H, S full Hermitian in (pinned) host memory.

    The fused public entry point equivalent to `compute_AB` followed by `build_all`
    (the reference CLI's regenerate flow, `cli.py:283-292`, `:310-325`), without the
    A*/B* round trip through host memory.  Pass a `pipeline` to reuse HBM buffers
    across k-points and `host_out=(H_pinned, S_pinned)` torch tensors to reuse pinned
    outputs."""
    from .builder import BuildConfig
    from .matrix import ComplexDense

    config = config or BuildConfig()
    dspec = DeviceSpec(spec)
    tpack = pack_tmats(tmats)
    pipe = pipeline or HSPipeline(spec.n_basis, dspec.heights)
    t = device.torch()
    n = spec.n_basis
    if host_out is None or tuple(host_out[0].shape) != (n, n):
        host_out = (t.empty((n, n), dtype=t.complex128, pin_memory=True),
                    t.empty((n, n), dtype=t.complex128, pin_memory=True))
    res = pipe.run(dspec, tpack, config.force_general_path, host_out=host_out)
    h = ComplexDense(host_out[0].numpy().T)
    s = ComplexDense(host_out[1].numpy().T)
    res["h2d_bytes"] = dspec.h2d_bytes + tpack.h2d_bytes
    res["d2h_bytes"] = 2 * 16 * n * n
    return h, s, res
