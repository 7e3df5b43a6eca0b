"""Frame-sharded multi-GPU rendering (BASELINE.json north_star).

The surfel set is replicated on every rank; sensor frames are sharded by
TIMESTEP in contiguous blocks (rank r renders timesteps [lo_r, hi_r), all
sensors of each), so each rank's frames are one contiguous slice of the
batch-ordered output and the only exchange step -- the final gather of the
frames to rank 0 -- lands every peer's slice directly in rank 0's output
slab with one point-to-point receive (NCCL over NVLink on GPUs, gloo in the
CPU tests).  No collective touches the data path before the gather, and
frames are never split across ranks (depth-ordered compositing does not
shard).  Contiguous blocks keep the camera/LiDAR mix identical per rank;
the street generator is uniform along the road, so per-timestep cost is
flat and blocks balance as well as a round-robin deal would.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None):
    """Initialise the default process group when WORLD_SIZE > 1.
    Returns (rank, world, device)."""
    rank, world, local = env_world()
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
    else:
        device = torch.device("cpu")
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        be = backend or ("nccl" if device.type == "cuda" else "gloo")
        kw = dict(backend=be, rank=rank, world_size=world)
        if be == "nccl":
            kw["device_id"] = device
            # communicator set-up lines (INIT subsystem only) to a per-process file, echoed
            # by nccl_init_info() so a run shows how many ranks the communicator joined
            if "NCCL_DEBUG" not in os.environ:
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
                os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(
                    os.environ.get("TMPDIR", "/tmp"), "gsr_nccl.%h.%p.log"))
        dist.init_process_group(**kw)
    return rank, world, device


def nccl_init_info(echo: bool = True):
    """This process's NCCL communicator set-up lines (NCCL_DEBUG_SUBSYS=INIT,
    written to NCCL_DEBUG_FILE by init()); echoed to stderr.  Returns
    {"nranks": [...], "init_complete": n, "lines": [...]} or None."""
    import glob
    import re
    import socket
    import sys
    pat = os.environ.get("NCCL_DEBUG_FILE")
    if not pat:
        return None
    path = pat.replace("%h", socket.gethostname()).replace("%p", str(os.getpid()))
    files = [path] if os.path.exists(path) else glob.glob(pat.replace("%h", "*").replace("%p", str(os.getpid())))
    lines = []
    for f in files:
        with open(f, errors="replace") as fh:
            lines += [ln.rstrip() for ln in fh if "Init COMPLETE" in ln or "nranks" in ln or "NCCL version" in ln]
    if echo:
        for ln in lines[:16]:
            print("[nccl]", ln, file=sys.stderr)
    nr = sorted({int(m) for ln in lines for m in re.findall(r"nranks (\d+)", ln)})
    return {"nranks": nr, "init_complete": sum("Init COMPLETE" in ln for ln in lines), "lines": lines[:8]}


def shard_range(n_items: int, world: int, rank: int):
    """Contiguous block [lo, hi) of n_items for `rank`; the first
    n_items % world ranks get one extra item."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_counts(n_items: int, world: int):
    return [shard_range(n_items, world, r)[1] - shard_range(n_items, world, r)[0] for r in range(world)]


def gather_blocks(local: torch.Tensor, full: torch.Tensor | None, n_items: int, world: int, rank: int,
                  root: int = 0, group=None):
    """Gather every rank's contiguous block of a batch (dim 0) into `full`
    on `root` with point-to-point transfers (one recv per peer into the
    peer's slice of `full`; the root's own block is copied unless `local`
    already is that slice).  `local` has shard_counts(...)[rank] rows.
    Returns the list of outstanding requests (wait() them, or let the
    caller's stream order them on NCCL)."""
    if world == 1:
        if full is not None and local.data_ptr() != full.data_ptr():
            full.copy_(local)
        return []
    ops = []
    if rank == root:
        assert full is not None and full.shape[0] == n_items
        for r in range(world):
            lo, hi = shard_range(n_items, world, r)
            if r == root:
                if local.data_ptr() != full[lo:hi].data_ptr() and hi > lo:
                    full[lo:hi].copy_(local)
            elif hi > lo:
                ops.append(dist.P2POp(dist.irecv, full[lo:hi], r, group))
    else:
        if local.shape[0] > 0:
            ops.append(dist.P2POp(dist.isend, local.contiguous(), root, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


def max_over_ranks(x: float, device, world: int) -> float:
    """Device-timed quantity -> its maximum over ranks."""
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int, device=None):
    if world > 1:
        if device is not None and device.type == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def round_ops(local: dict, full: dict | None, j: int, n_items: int, world: int, rank: int, root: int = 0,
              group=None):
    """Point-to-point ops of gather round j: every non-root rank sends the j-th
    item of its block (one tensor per key of `local`, e.g. the camera and the
    LiDAR frames of its j-th timestep) and the root receives item j of every
    peer's block straight into its slot of `full`.  All ranks issue the rounds
    in the same order, so each round's sends and receives match one to one;
    posting round j as soon as item j is rendered overlaps the transfer with
    the rendering of the next items."""
    ops = []
    if world == 1:
        return ops
    if rank == root:
        for r in range(world):
            if r == root:
                continue
            lo, hi = shard_range(n_items, world, r)
            if j < hi - lo:
                for k in sorted(full):
                    ops.append(dist.P2POp(dist.irecv, full[k][lo + j], r, group))
    else:
        lo, hi = shard_range(n_items, world, rank)
        if j < hi - lo:
            for k in sorted(local):
                ops.append(dist.P2POp(dist.isend, local[k][j], root, group))
    return ops


def n_rounds(n_items: int, world: int) -> int:
    return max(shard_counts(n_items, world)) if world > 0 else 0


class ShardedBatch:
    """Output layout and gather of a frame-sharded batch (the bookkeeping of
    bench.py's multi-GPU step).  The batch is n_t timesteps with the same
    frames each (`frame_specs`: (kind, C, H, W) per frame of a timestep);
    this rank renders timesteps [lo, hi) (shard_range).  Frames are stored in
    one slab per kind in batch order: rank 0 allocates the whole batch
    (`full`) and renders straight into its own slice, the other ranks hold
    only their block (`local`).  `outs[i]` is the tensor local frame i (in
    timestep-major order) is rendered into.  The only exchange is the gather
    to rank 0: all at the end (`gather`) or one timestep round at a time
    (`round`), overlapping the rendering of the next timesteps."""

    def __init__(self, frame_specs, n_t: int, world: int, rank: int, device, dtype=torch.float32):
        self.specs = list(frame_specs)
        self.n_t, self.world, self.rank = n_t, world, rank
        self.lo, self.hi = shard_range(n_t, world, rank)
        self.kinds = sorted({int(k) for k, *_ in self.specs})
        self.per_t = {k: sum(1 for s in self.specs if int(s[0]) == k) for k in self.kinds}
        self.full, self.local = {}, {}
        nloc = self.hi - self.lo
        for k in self.kinds:
            _, C, H, W = next(s for s in self.specs if int(s[0]) == k)
            if rank == 0:
                self.full[k] = torch.empty((n_t * self.per_t[k], C, H, W), dtype=dtype, device=device)
                self.local[k] = self.full[k][self.per_t[k] * self.lo: self.per_t[k] * self.hi]
            else:
                self.local[k] = torch.empty((nloc * self.per_t[k], C, H, W), dtype=dtype, device=device)
        self.outs = []
        for j in range(nloc):
            seen = {k: 0 for k in self.kinds}
            for kind, *_ in self.specs:
                k = int(kind)
                self.outs.append(self.local[k][j * self.per_t[k] + seen[k]])
                seen[k] += 1
        self.local_blocks = {k: self.local[k].view(nloc, self.per_t[k], *self.local[k].shape[1:])
                             for k in self.kinds}
        self.full_blocks = ({k: self.full[k].view(n_t, self.per_t[k], *self.full[k].shape[1:])
                             for k in self.kinds} if rank == 0 else None)

    @property
    def frames_per_timestep(self) -> int:
        return len(self.specs)

    def gather(self):
        """Gather every rank's block to rank 0 (point-to-point), and wait."""
        if self.world == 1:
            return
        reqs = []
        for k in self.kinds:
            fv = self.full_blocks[k] if self.full_blocks is not None else None
            reqs += gather_blocks(self.local_blocks[k], fv, self.n_t, self.world, self.rank)
        for r in reqs:
            r.wait()

    def round(self, j: int):
        """Post gather round j (item j of every rank's block); returns the requests."""
        ops = round_ops(self.local_blocks, self.full_blocks, j, self.n_t, self.world, self.rank)
        return dist.batch_isend_irecv(ops) if ops else []

    def rounds_left(self):
        """Rounds rank 0 still has to receive after posting one per own timestep
        (uneven blocks: peers with more timesteps than the root)."""
        return range(self.hi - self.lo, n_rounds(self.n_t, self.world)) if self.rank == 0 else range(0)
