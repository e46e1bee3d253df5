"""Device-resident H/S setup pipeline (the B200 hot path).

    SystemSpec + T blocks --(H2D, tiny)--> [A/B generator] --> [native build] --> H, S

`HSPipeline` owns the HBM buffers for one problem shape and runs one k-point per
call as a single native call (`hsdla_setup_hs`): the fused A/B generator (reference
`flapw.py:201-233`) writes A, B and the row-scaled B, the T preparation / Cholesky runs
on a side stream meanwhile, then the T-block applications and the two triangular DMMA
contractions with the Hermitian mirror fused into their epilogue (reference
`builder.py:403-474`).  Inputs stay resident; only the spec, the T blocks and (when
asked) the results cross PCIe.  `run_async` / `finish` pipeline consecutive k-points:
the D2H copies of k-point i overlap the compute of k-point i+1.

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


_UPLOAD = {}


_TORCH_DTYPE = {}  # numpy dtype string -> torch dtype (filled on first use)


def _to_device(arrays):
    """Upload host arrays through pinned staging on a dedicated upload stream, so the
    copies run at once instead of queueing behind kernels already enqueued on the compute
    stream (k-point pipelining); the compute stream waits on an event.  Returns (device
    tensors, pinned staging tensors that must stay alive until the copies ran)."""
    t = device.torch()
    if not _TORCH_DTYPE:
        _TORCH_DTYPE.update({"<f8": t.float64, "<c16": t.complex128, "<i4": t.int32,
                             "<i8": t.int64})
    dev = t.cuda.current_device()
    up = _UPLOAD.get(dev)
    if up is None:
        up = _UPLOAD[dev] = t.cuda.Stream()
    main = t.cuda.current_stream()
    # one pinned staging buffer and one copy for all of them (each array's bytes at a
    # 256-byte aligned offset); the device tensors are typed views of one allocation
    arrays = [np.ascontiguousarray(a) for a in arrays]
    offs, n = [], 0
    for a in arrays:
        offs.append(n)
        n += (a.nbytes + 255) // 256 * 256
    staged = t.empty(max(n, 1), dtype=t.uint8, pin_memory=True)
    host = staged.numpy()
    for a, o in zip(arrays, offs):
        host[o:o + a.nbytes] = a.reshape(-1).view(np.uint8)
    with t.cuda.stream(up):
        whole = staged.to("cuda", non_blocking=True)
        done = t.cuda.Event()
        done.record(up)
    main.wait_event(done)
    whole.record_stream(main)
    out = [whole[o:o + a.nbytes].view(_TORCH_DTYPE[a.dtype.str]).view(a.shape)
           for a, o in zip(arrays, offs)]
    return out, staged


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
    _staging: object = None
    t_dense: np.ndarray = None  # (n_tsets,) int32: (l_nonsph+1)^2 dense-block size per set

    @property
    def n_tsets(self) -> int:
        return int(self.t_dim.shape[0])


def tset_udot2(tpack, heights, row_offset, udot_rows) -> np.ndarray:
    """(n_tsets, max t_dim) ||udot||^2 rows per T set for the shifted joint form; a row of -1
    where the set's atoms differ in ||udot|| or have T smaller than their block (no shift)."""
    mp = int(max(1, int(np.max(tpack.t_dim))))
    out = np.full((tpack.n_tsets, mp), -1.0)
    u = np.asarray(udot_rows, dtype=np.float64)
    for t in range(tpack.n_tsets):
        m = int(tpack.t_dim[t])
        atoms = np.nonzero(np.asarray(tpack.t_index) == t)[0]
        rows = [u[int(row_offset[a]):int(row_offset[a]) + int(heights[a])] for a in atoms]
        if rows and all(len(r) == m for r in rows) and all(np.array_equal(r, rows[0]) for r in rows):
            out[t, :m] = rows[0] * rows[0]
    return out


def pack_tmats(tmats) -> TPack:
    """Deduplicate per-atom T blocks by identity and upload them (one H2D)."""
    device.require_cuda()
    keys, index, reps = {}, [], []
    for a in range(tmats.atom_count):
        key = (id(tmats.t_aa[a]), id(tmats.t_ab[a]), id(tmats.t_bb[a]))
        if key not in keys:
            keys[key] = len(reps)
            reps.append(a)
        index.append(keys[key])
    dims = np.array([tmats.t_aa[a].rows for a in reps], dtype=np.int32)
    l_ns = getattr(tmats, "l_nonsph", None)
    dense = np.array([min(int(dims[s]), (int(l_ns[a]) + 1) ** 2) if l_ns is not None
                      and a < len(l_ns) else int(dims[s]) for s, a in enumerate(reps)],
                     dtype=np.int32)
    t_ld = int(max(1, dims.max()))
    host = np.zeros((3, len(reps), t_ld, t_ld), dtype=np.complex128)
    for s, a in enumerate(reps):
        m = int(dims[s])
        for f, fam in enumerate((tmats.t_aa, tmats.t_ab, tmats.t_bb)):
            host[f, s, :m, :m] = fam[a].array.T  # (col, row) storage = column-major
    index = np.array(index, dtype=np.int32)
    # Content cache: the same T values (any objects) on the same device reuse the uploaded pack,
    # so repeated single calls keep the pipeline's cached T preparation (reuse_t); a T changed
    # in place compares unequal and is uploaded afresh.
    dev_id = device.torch().cuda.current_device()
    hit = _TPACK_CACHE.get(dev_id)
    if (hit is not None and hit[0].shape == host.shape and np.array_equal(hit[1], index)
            and np.array_equal(hit[2], dense) and np.array_equal(hit[3].t_dim, dims)
            and np.array_equal(hit[0], host)):
        return hit[3]
    (dev,), staged = _to_device([host])
    pack = TPack(index, dims, t_ld, dev[0], dev[1], dev[2], host.nbytes, staged, dense)
    _TPACK_CACHE[dev_id] = (host, index.copy(), dense, pack)
    return pack


_TPACK_CACHE: dict = {}  # device -> (packed host T, t_index, t_dense, TPack) of the last pack


class DeviceSpec:
    """A SystemSpec's arrays in HBM (k-vectors, positions, rotations, radii, radial table)."""

    def __init__(self, spec):
        device.require_cuda()
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
            radial[a, :n] = np.stack((rad.u[:n], rad.u_prime[:n], rad.udot[:n], rad.udot_prime[:n],
                                      rad.udot_norm[:n]), axis=-1)
        self.radial_stride = stride
        # ||udot|| per stacked row (l^2 + l + m order): the joint form's shift metric
        self.udot_rows = np.concatenate([np.repeat(np.asarray(spec.radial[a].udot_norm[:l + 1], dtype=np.float64),
                                                   2 * np.arange(l + 1) + 1)
                                         for a, l in enumerate(self.l_sph)])
        host = [np.asarray(spec.k_vectors, dtype=np.float64),
                np.asarray(spec.positions, dtype=np.float64),
                np.asarray(spec.rotations, dtype=np.float64).reshape(-1, 9),
                np.asarray(spec.mt_radius, dtype=np.float64), radial]
        # Atom types of the template path (hsdla_build_args.atom_type): atoms with identical
        # rotation, muffin-tin radius, l_sph and radial data (exact equality) share one type;
        # _Call refines them by T set.
        keys, types = {}, []
        for a in range(self.n_atoms):
            key = (host[2][a].tobytes(), host[3][a].tobytes(), int(self.l_sph[a]),
                   radial[a].tobytes())
            types.append(keys.setdefault(key, len(keys)))
        self.atom_type = np.asarray(types, dtype=np.int32)
        self.h2d_bytes = int(sum(h.nbytes for h in host))
        dev, self._staging = _to_device(host)
        self.kv, self.pos, self.rot, self.rmt, self.radial = dev
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
    args.l_sph = dspec.l_sph.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.row_offset = dspec.row_offset.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
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


class _Call:
    """Argument blocks of one native build call (kept alive while it is in flight)."""

    def __init__(self, *, n_basis, heights, row_offset, tpack: TPack, A, B, Bs, udot, ld,
                 force_general_path, H, S, ldh, shard_rank, n_shards, workspace, host_out,
                 ab_args=None, shard_mirror=False, reuse_t=False, stream_h_copy=0,
                 h_reference_form=False, host_src=None, n_capacity=None, udot_rows=None,
                 atom_type=None):
        lib = _native.load()
        t = device.torch()
        self.na = len(heights)
        self.n_tsets = tpack.n_tsets
        self.keep = [np.ascontiguousarray(heights, dtype=np.int32),
                     np.ascontiguousarray(row_offset, dtype=np.int64),
                     np.ascontiguousarray(tpack.t_index, dtype=np.int32),
                     np.ascontiguousarray(tpack.t_dim, dtype=np.int32), tpack, host_out, ab_args,
                     np.ascontiguousarray(tpack.t_dense if tpack.t_dense is not None
                                          else tpack.t_dim, dtype=np.int32)]
        h_arr, o_arr, ti, td = self.keep[:4]
        a = _native.BuildArgs()
        a.n_atoms = self.na
        a.n_basis = n_basis
        a.heights = h_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        a.row_offset = o_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        a.t_index = ti.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        a.n_tsets = tpack.n_tsets
        a.t_dim = td.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        a.t_dense = self.keep[-1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        if atom_type is not None:
            pairs, typed = {}, []
            for ty, ts in zip(np.asarray(atom_type), np.asarray(tpack.t_index)):
                typed.append(pairs.setdefault((int(ty), int(ts)), len(pairs)))
            at = np.asarray(typed, dtype=np.int32)
            self.keep.append(at)
            a.atom_type = at.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            a.n_types = len(pairs)
        if udot_rows is not None and n_shards <= 1:
            u2 = tset_udot2(tpack, heights, row_offset, udot_rows)
            self.keep.append(u2)
            a.t_udot2 = u2.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        a.t_aa = tpack.t_aa.data_ptr()
        a.t_ab = tpack.t_ab.data_ptr()
        a.t_bb = tpack.t_bb.data_ptr()
        a.t_ld = tpack.t_ld
        a.A = A.data_ptr()
        a.B = B.data_ptr()
        a.B_scaled = Bs.data_ptr() if Bs is not None else None
        a.udot_norms = udot.data_ptr() if udot is not None else None
        a.ld = ld
        a.force_general_path = 1 if force_general_path else 0
        a.H = H.data_ptr()
        a.S = S.data_ptr()
        a.ldh = ldh
        a.shard_rank = shard_rank
        a.n_shards = n_shards
        a.shard_mirror = 1 if shard_mirror else 0
        a.reuse_t = 1 if reuse_t else 0
        a.stream_h_copy = int(stream_h_copy)
        a.h_reference_form = 1 if h_reference_form else 0
        if host_src is not None:  # (A_host ptr, B_host ptr, ld): pinned sources the build uploads
            a.A_host, a.B_host, a.ld_ab_host = host_src
        if host_out is not None:  # pinned (n, n) tensors, row j = column j
            a.H_host = host_out[0].data_ptr()
            a.S_host = host_out[1].data_ptr()
            a.ldh_host = int(host_out[0].shape[1])
        self.need = lib.hsdla_build_workspace_size(ctypes.byref(a))
        if workspace is None or workspace.numel() < self.need:
            # size for the caller's capacity (a k-point batch with varying N_G keeps one
            # workspace, so its T preparation stays reusable)
            a.n_basis = max(n_basis, int(n_capacity or 0))
            cap_need = lib.hsdla_build_workspace_size(ctypes.byref(a))
            a.n_basis = n_basis
            workspace = t.empty(max(self.need, cap_need, 1), dtype=t.uint8, device="cuda")
        self.workspace = workspace
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = workspace.numel()
        self.args = a
        self.ab = ab_args
        self.mask = (ctypes.c_int32 * self.na)()
        self.info = (ctypes.c_int32 * self.n_tsets)()
        self.res = _native.BuildResult()
        self.joint = (ctypes.c_int32 * self.n_tsets)()
        self.res.hpd_mask = self.mask
        self.res.chol_info = self.info
        self.res.joint_info = self.joint

    def result(self, rc: int) -> dict:
        if rc == _native.HSDLA_ERR_NAN_INPUT:
            raise ContractViolationError("NaN in Cholesky input (lower triangle)")
        if rc == _native.HSDLA_ERR_NONFINITE:
            raise ContractViolationError("accumulator contains non-finite values")
        _native.check(rc, "hsdla_build_hs")
        r = self.res
        return {
            "hpd_mask": [bool(self.mask[i]) for i in range(self.na)],
            "chol_info": [int(self.info[i]) for i in range(self.n_tsets)],
            "joint_t": [bool(self.joint[i]) for i in range(self.n_tsets)],
            "joint_split": [self.joint[i] == 2 for i in range(self.n_tsets)],
            "joint_shift": float(r.joint_shift),
            "template_types": int(r.template_types),
            "ms_templates": float(r.ms_templates),
            "merged_sh": bool(r.merged_sh),
            "ms": {"setup": r.ms_setup, "S": r.ms_S, "H_ABBA_BB": r.ms_H_ABBA_BB,
                   "H_AA": r.ms_H_AA},
            # template path: the per-type W = L^H [A; B] application and the W1 / W2 expansion
            "kernel_ms": ({"contract_S": r.ms_contract_S, "contract_H": r.ms_contract_H,
                           "apply_W": r.ms_apply_Z, "expand_W": r.ms_apply_XY}
                          if r.template_types and all(self.joint[i] == 1 for i in range(self.n_tsets))
                          else {"contract_S": r.ms_contract_S, "contract_H": r.ms_contract_H,
                                "apply_Z": r.ms_apply_Z, "apply_XY": r.ms_apply_XY}),
            "workspace_bytes": int(self.need),
            "ms_total": r.ms_total,
        }

    def run_sync(self) -> dict:
        lib = _native.load()
        if self.ab is not None:
            rc = lib.hsdla_setup_hs(device.ctx(), ctypes.byref(self.ab), ctypes.byref(self.args),
                                    ctypes.byref(self.res))
        else:
            rc = lib.hsdla_build_hs(device.ctx(), ctypes.byref(self.args), ctypes.byref(self.res))
        return self.result(rc)

    def start(self) -> int:
        lib = _native.load()
        ticket = ctypes.c_ulonglong(0)
        ab = ctypes.byref(self.ab) if self.ab is not None else None
        _native.check(lib.hsdla_setup_hs_async(device.ctx(), ab, ctypes.byref(self.args),
                                               ctypes.byref(ticket)), "hsdla_setup_hs_async")
        return ticket.value

    def finish(self, ticket: int) -> dict:
        rc = _native.load().hsdla_build_finish(device.ctx(), ctypes.c_ulonglong(ticket),
                                               ctypes.byref(self.res))
        return self.result(rc)


def build_device(*, n_basis, heights, row_offset, tpack: TPack, A, B, Bs, udot, ld,
                 force_general_path, H, S, ldh, shard_rank=0, n_shards=1, workspace=None,
                 ab_args=None, host_out=None, h_reference_form=False, host_src=None,
                 udot_rows=None, reuse_t=False):
    """Synchronous `hsdla_build_hs` (or `hsdla_setup_hs` when `ab_args` is given: A/B
    generation fused in front); returns (result dict, workspace tensor).  `reuse_t`: the T
    pack is the one the previous build on this `workspace` used (its T preparation is kept)."""
    call = _Call(n_basis=n_basis, heights=heights, row_offset=row_offset, tpack=tpack, A=A, B=B,
                 Bs=Bs, udot=udot, ld=ld, force_general_path=force_general_path, H=H, S=S,
                 ldh=ldh, shard_rank=shard_rank, n_shards=n_shards, workspace=workspace,
                 host_out=host_out, ab_args=ab_args, reuse_t=reuse_t,
                 h_reference_form=h_reference_form, host_src=host_src, udot_rows=udot_rows)
    return call.run_sync(), call.workspace


class HSPipeline:
    """Reusable HBM buffers for up to `n_capacity` basis functions and one atom layout;
    `run` = one k-point (any N_G <= n_capacity, e.g. a k-point batch with varying G-sets)."""

    def __init__(self, n_capacity: int, heights, *, shard_rank: int = 0, n_shards: int = 1,
                 out=None, shard_mirror: bool = False, h_reference_form: bool = False):
        """`out` = (H, S) device (n_capacity, ld) tensors to write instead of own buffers
        (e.g. a peer rank's, mapped through NVLink); `shard_mirror`, `h_reference_form` see
        hsdla_build_args (the latter: always the reference's Z / Y forms for H instead of the
        joint factor of the per-type T matrix)."""
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
        if out is None:
            self.H = device.empty_matrix(n, n, n)
            self.S = device.empty_matrix(n, n, n)
        else:
            self.H, self.S = out
            if tuple(self.H.shape) != (n, n) or tuple(self.S.shape) != (n, n):
                raise ContractViolationError("output buffers must be (n_capacity, n_capacity)")
        self._own_out = out is None
        self._alt = None  # second device (H, S) pair for pipelined k-points (run_async)
        self._flip = 0
        self.workspace = None
        self.shard_rank, self.n_shards = shard_rank, n_shards
        self.shard_mirror = bool(shard_mirror)
        self.h_reference_form = bool(h_reference_form)
        self._last_t = None  # (TPack, force) of the previous call: T forms reusable
        self.n_basis = 0
        self._inflight = {}

    @property
    def device_bytes(self) -> int:
        tot = sum(x.numel() * x.element_size() for x in (self.A, self.B, self.Bs, self.udot,
                                                          self.H, self.S))
        if self._alt is not None:
            tot += sum(x.numel() * x.element_size() for x in self._alt)
        if self.workspace is not None:
            tot += self.workspace.numel()
        return int(tot)

    def _call(self, dspec: DeviceSpec, tpack: TPack, force_general_path: bool, host_out,
              stream_h_copy: int = 0, alternate: bool = False):
        if dspec.n_basis > self.n_capacity or dspec.rows != self.rows:
            raise ContractViolationError("spec shape does not fit the pipeline buffers")
        self.n_basis = dspec.n_basis
        ab = make_ab_args(dspec, self.A, self.B, self.Bs, self.ld, None)
        # A TPack is an immutable device copy, so the same object means the same T: its
        # forms and Cholesky factors from the previous call are still in the workspace.
        last = self._last_t
        reuse = last is not None and last[0] is tpack and last[1] == bool(force_general_path)
        H, S = self.H, self.S
        if alternate and self._own_out and host_out is not None:
            # Pipelined k-points with host copies alternate two device (H, S) pairs, so
            # k-point i+1's contractions never wait for k-point i's copies (hsdla_setup_hs_async).
            if self._alt is None:
                n = self.n_capacity
                self._alt = (device.empty_matrix(n, n, n), device.empty_matrix(n, n, n))
            if self._flip:
                H, S = self._alt
            self._flip ^= 1
        self._last_out = (H, S)
        call = _Call(n_basis=dspec.n_basis, heights=dspec.heights, row_offset=dspec.row_offset,
                     tpack=tpack, A=self.A, B=self.B, Bs=self.Bs, udot=self.udot, ld=self.ld,
                     force_general_path=force_general_path, H=H, S=S,
                     ldh=self.n_capacity, shard_rank=self.shard_rank, n_shards=self.n_shards,
                     workspace=self.workspace, host_out=host_out, ab_args=ab,
                     shard_mirror=self.shard_mirror, reuse_t=reuse, stream_h_copy=stream_h_copy,
                     h_reference_form=self.h_reference_form, n_capacity=self.n_capacity,
                     udot_rows=dspec.udot_rows, atom_type=dspec.atom_type)
        call.keep.append(dspec)
        self.workspace = call.workspace
        self._last_t = (tpack, bool(force_general_path))
        return call

    def run(self, dspec: DeviceSpec, tpack: TPack, force_general_path: bool = False,
            host_out=None) -> dict:
        """One k-point, spec -> H, S in HBM (and in `host_out` pinned (n, n) tensors when
        given), as a single synchronous native call (`hsdla_setup_hs`)."""
        return self._call(dspec, tpack, force_general_path, host_out).run_sync()

    def run_async(self, dspec: DeviceSpec, tpack: TPack, force_general_path: bool = False,
                  host_out=None, last: bool = False) -> int:
        """Enqueue one k-point and return a ticket at once (`hsdla_setup_hs_async`).  At
        most two k-points may be in flight; their `host_out` buffers must differ.  `last`:
        no k-point follows, so H is streamed to the host during its own contraction."""
        call = self._call(dspec, tpack, force_general_path, host_out, 1 if last else 0,
                          alternate=True)
        ticket = call.start()
        self._inflight[ticket] = call
        return ticket

    def finish(self, ticket: int) -> dict:
        """Wait for a k-point enqueued by `run_async` (compute and host copies)."""
        return self._inflight.pop(ticket).finish(ticket)

    def launches_per_run(self, dspec: DeviceSpec, result: dict | None = None) -> int:
        """Kernels this pipeline launches per k-point once the T preparation is cached.
        Per-atom path: A/B per l group, S contraction, Z apply, XY apply, H contraction, result
        publication (plus the tail kernel of split T sets, which the caller adds from
        `joint_split`).  Template path (`result["template_types"] > 0`): templates per l group,
        expansion, S contraction, per-type W application, W expansion, H contraction,
        publication; merged (`result["merged_sh"]`): S and H are one contraction launch."""
        groups = len(np.unique(dspec.l_sph))
        if result is not None and result.get("template_types", 0) and "apply_W" in result.get(
                "kernel_ms", {}):
            return groups + (5 if result.get("merged_sh") else 6)
        return groups + 5

    def result_views(self):
        """Host-indexable (n, n) views: H[i, j] == tensor[j, i] (column-major storage)."""
        n = self.n_basis
        h, s = getattr(self, "_last_out", (self.H, self.S))
        return h[:n, :n], s[:n, :n]


def _pinned_pair(n: int):
    t = device.torch()
    return (t.empty((n, n), dtype=t.complex128, pin_memory=True),
            t.empty((n, n), dtype=t.complex128, pin_memory=True))


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
    n = spec.n_basis
    if host_out is None or tuple(host_out[0].shape) != (n, n):
        host_out = _pinned_pair(n)
    res = pipe.run(dspec, tpack, config.force_general_path, host_out=host_out)
    res["h2d_bytes"] = dspec.h2d_bytes + tpack.h2d_bytes
    res["d2h_bytes"] = 2 * 16 * n * n
    return ComplexDense(host_out[0].numpy().T), ComplexDense(host_out[1].numpy().T), res


def build_hs_many(specs, tmats, config=None, *, pipeline: HSPipeline | None = None,
                  on_result=None, host_buffers=None):
    """A k-point batch (same crystal, T blocks shared): H and S of every k-point land in
    pinned host memory, with k-point i's D2H copies overlapping k-point i+1's compute.

    `on_result(index, H, S, result)` is called for each k-point as soon as it is complete
    (H, S are `ComplexDense` views of double-buffered pinned memory, valid until the
    callback returns).  Every k-point uploads its own spec (H2D) and T blocks are uploaded
    once per batch.  Returns the list of result dicts."""
    from .builder import BuildConfig
    from .matrix import ComplexDense

    config = config or BuildConfig()
    specs = list(specs)
    if not specs:
        return []
    n_cap = max(s.n_basis for s in specs)
    tpack = pack_tmats(tmats)
    first = DeviceSpec(specs[0])
    pipe = pipeline or HSPipeline(n_cap, first.heights)
    bufs = host_buffers if host_buffers is not None else {}
    results = []
    pending = None  # (index, ticket, host_out, dspec)
    for i, spec in enumerate(specs):
        dspec = first if i == 0 else DeviceSpec(spec)
        n = spec.n_basis
        key = (i % 2, n)
        if key not in bufs:
            bufs[key] = _pinned_pair(n)
        ticket = pipe.run_async(dspec, tpack, config.force_general_path, host_out=bufs[key],
                                last=(i == len(specs) - 1))
        if pending is not None:
            results.append(_complete(pipe, pending, tpack, on_result, ComplexDense))
        pending = (i, ticket, bufs[key], dspec)
    results.append(_complete(pipe, pending, tpack, on_result, ComplexDense))
    return results


def _complete(pipe, pending, tpack, on_result, ComplexDense):
    i, ticket, host_out, dspec = pending
    res = pipe.finish(ticket)
    n = dspec.n_basis
    res["h2d_bytes"] = dspec.h2d_bytes + (tpack.h2d_bytes if i == 0 else 0)
    res["d2h_bytes"] = 2 * 16 * n * n
    if on_result is not None:
        on_result(i, ComplexDense(host_out[0].numpy().T), ComplexDense(host_out[1].numpy().T), res)
    return res
