"""Multi-GPU partitioning of the H/S setup.

Two ways, one process per GPU (torch.distributed, NCCL over NVLink on the box):

* **k-points** — independent; rank r builds k-points r, r+P, ...; no collective in the
  data path (`kpoints_for_rank`).
* **column panels of one large k-point** — every rank regenerates A*, B*, Z, XY locally
  from the tiny spec + T (cheaper than broadcasting GBs), computes the lower tiles of the
  64-wide column panels it owns (`hsdla_build_args.shard_rank / n_shards`), and the
  panels are gathered to one consumer rank with point-to-point sends; the consumer writes
  the Hermitian mirror.  Each tile's full K-sum is local, so no reduction is needed.
  Panel j and panel nb-1-j form one balanced pair (their lower-triangle tile counts sum
  to nb+1); pairs are dealt round-robin (`panel_owner`, the same rule as the C ABI's
  `hsdla_panel_owner`).
"""
from __future__ import annotations

PANEL = 64  # column panel width = the contraction tile edge


def panel_owner(n_panels: int, n_shards: int, panel: int) -> int:
    """Owner rank of a column panel (restates `hsdla_panel_owner`, csrc/capi.cu)."""
    if n_shards <= 1:
        return 0
    return min(panel, n_panels - 1 - panel) % n_shards


def owned_panels(n: int, n_shards: int, rank: int) -> list:
    nb = (n + PANEL - 1) // PANEL
    return [j for j in range(nb) if panel_owner(nb, n_shards, j) == rank]


def panel_tiles(n: int, panel: int) -> int:
    """Lower-triangle 64x64 tiles in column panel `panel`."""
    nb = (n + PANEL - 1) // PANEL
    return nb - panel


def kpoints_for_rank(n_kpoints: int, n_shards: int, rank: int) -> list:
    """Round-robin k-point assignment (C5: 64 k-points over 1/2/4/8 GPUs)."""
    return list(range(rank, n_kpoints, n_shards))


def gather_panels(mat, n: int, world: int, rank: int, dst: int = 0, group=None):
    """Gather owned column panels of a column-major matrix to rank `dst`, in place.

    `mat` is a (n_cols, ld) tensor whose row j holds column j (the layout of every device
    matrix here), so column panel [j0, j0+64) is the contiguous slice mat[j0:j0+64].  Each
    rank sends the panels it owns; `dst` receives the others straight into place.  Works
    with NCCL (GPU tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    nb = (n + PANEL - 1) // PANEL
    # gloo moves host memory only: device panels are staged through host copies (the NCCL
    # path on the GPU box sends device memory directly)
    staged = mat.is_cuda and dist.get_backend(group) == "gloo"
    # complex panels travel as their float64 (re, im) view: NCCL's point-to-point calls take
    # real data types only
    real = torch.view_as_real(mat) if mat.is_complex() else mat
    ops, back = [], []
    for j in range(nb):
        owner = panel_owner(nb, world, j)
        sl = real[j * PANEL:min(n, (j + 1) * PANEL)]
        if rank == dst and owner != dst:
            buf = sl.cpu() if staged else sl
            ops.append(dist.P2POp(dist.irecv, buf, owner, group))
            if staged:
                back.append((sl, buf))
        elif rank == owner and owner != dst:
            ops.append(dist.P2POp(dist.isend, sl.cpu() if staged else sl, dst, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for dev, host in back:
        dev.copy_(host)
    return mat


def _group_info(group):
    """(world, rank) of `group`; (1, 0) without an initialised process group."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


class NcclShardedBuild:
    """Reusable state of the NCCL panel-sharded build of one k-point shape: every rank owns
    an HSPipeline that computes the lower tiles of its column panels; `run` gathers the
    panels to `dst` (batched send/recv, `gather_panels`) and mirrors there.  Works without
    a process group (one rank: the plain build plus the mirror pass)."""

    def __init__(self, n: int, heights, *, dst: int = 0, group=None):
        from .pipeline import HSPipeline

        self.group = group
        self.world, self.rank = _group_info(group)
        self.dst = dst
        self.n = n
        self.pipe = HSPipeline(n, heights, shard_rank=self.rank, n_shards=self.world)

    def run(self, dspec, tpack, force_general_path: bool = False):
        """All ranks: build + gather; returns (H, S, result) device views on dst, None elsewhere."""
        import ctypes

        from . import _native, device
        from .errors import ContractViolationError

        n = self.n
        res = self.pipe.run(dspec, tpack, force_general_path)
        self.last_result = res
        if self.world > 1:
            gather_panels(self.pipe.H, n, self.world, self.rank, self.dst, self.group)
            gather_panels(self.pipe.S, n, self.world, self.rank, self.dst, self.group)
            if self.rank != self.dst:
                return None
            lib = _native.load()
            for m in (self.pipe.H, self.pipe.S):
                flag = ctypes.c_int32(0)
                _native.check(lib.hsdla_mirror_lower(device.ctx(), n, device.ptr(m), m.shape[1],
                                                     ctypes.byref(flag)), "hsdla_mirror_lower")
                if flag.value:
                    raise ContractViolationError("accumulator contains non-finite values")
        return self.pipe.H[:n, :n], self.pipe.S[:n, :n], res


def build_hs_sharded(spec, tmats, config=None, *, dst: int = 0, group=None,
                     transport: str = "nccl"):
    """One k-point's H and S computed by all ranks of the process group (column panels),
    assembled on rank `dst`; returns device (H, S, result) on `dst`, None elsewhere.
    Every rank must call it (collective).

    transport="nccl": each rank writes its panels locally, then `gather_panels` moves them
    to `dst` (batched NCCL send/recv) and `dst` runs the Hermitian mirror.
    transport="p2p": H and S live in symmetric memory; every rank's contraction epilogue
    stores its owned tiles and their conjugate mirror straight into `dst`'s buffers over
    NVLink (hsdla_build_args.shard_mirror), so compute and gather are one kernel and no
    mirror pass is left."""
    if transport == "p2p":
        return _build_hs_sharded_p2p(spec, tmats, config, dst=dst, group=group)
    if transport != "nccl":
        raise ValueError(f"unknown transport {transport!r}")
    from .builder import BuildConfig
    from .pipeline import DeviceSpec, pack_tmats

    config = config or BuildConfig()
    dspec = DeviceSpec(spec)
    return NcclShardedBuild(spec.n_basis, dspec.heights, dst=dst, group=group).run(
        dspec, pack_tmats(tmats), config.force_general_path)


class P2PShardedBuild:
    """Reusable state of the P2P panel-sharded build of one k-point shape: H and S in torch
    symmetric memory (mapped into every rank), the consumer's buffers as every rank's
    output, and an HSPipeline per rank writing its owned tiles + mirror there."""

    def __init__(self, n: int, heights, *, dst: int = 0, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        from .pipeline import HSPipeline

        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.dst = dst
        self.n = n
        self.local = [symm_mem.empty((n, n), dtype=torch.complex128, device="cuda")
                      for _ in range(2)]
        peers = []
        for buf in self.local:
            hdl = symm_mem.rendezvous(buf, self.group.group_name)
            peers.append(hdl.get_buffer(dst, (n, n), torch.complex128))
        self.pipe = HSPipeline(n, heights, shard_rank=self.rank, n_shards=self.world,
                               out=tuple(peers), shard_mirror=True)

    def run(self, dspec, tpack, force_general_path: bool = False):
        """All ranks: build; returns (H, S, result) device views on dst, None elsewhere."""
        import torch
        import torch.distributed as dist

        from .errors import ContractViolationError

        # Nobody stores into dst's H / S before dst has released the previous result (the
        # views returned by the last run stay valid until the next collective call).
        dist.barrier(group=self.group)
        try:
            res, bad = self.pipe.run(dspec, tpack, force_general_path), 0
        except ContractViolationError:
            res, bad = None, 1
        self.last_result = res
        torch.cuda.synchronize()  # this rank's remote stores are complete
        flag = torch.tensor([bad], device="cuda")
        dist.all_reduce(flag, group=self.group)  # orders every rank's stores before dst reads
        if int(flag.item()):
            raise ContractViolationError("accumulator contains non-finite values")
        if self.rank != self.dst:
            return None
        return self.local[0], self.local[1], res


def _build_hs_sharded_p2p(spec, tmats, config=None, *, dst: int = 0, group=None):
    from .builder import BuildConfig
    from .pipeline import DeviceSpec, pack_tmats

    config = config or BuildConfig()
    dspec = DeviceSpec(spec)
    return P2PShardedBuild(spec.n_basis, dspec.heights, dst=dst, group=group).run(
        dspec, pack_tmats(tmats), config.force_general_path)
