"""Multi-GPU plumbing: candidates shard across ranks by contiguous S* ranges (no
data-path collective); the single exchange is an all-reduce MIN of the packed
per-budget (cost << idx_bits | idx) keys.  torch.distributed
supplies the process group (NCCL over NVLink on GPUs, gloo in CPU tests)."""
from __future__ import annotations


def shard_range(n_sstar_total: int, rank: int, world: int):
    """Rank r owns S* [floor(r N / P), floor((r+1) N / P))."""
    lo = (rank * n_sstar_total) // world
    hi = ((rank + 1) * n_sstar_total) // world
    return lo, hi


def global_best(best_key, group=None):
    """In-place all-reduce MIN of the int64 keys; equal keys cannot come from two ranks
    because the index field is global, so the result is the global (cost, idx) argmin.
    The max-batch keys ((2^31-1 - B_max) << idx_bits | idx) reduce the same way."""
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        with torch.cuda.nvtx.range("cm_allreduce_min"):
            dist.all_reduce(best_key, op=dist.ReduceOp.MIN, group=group)
    return best_key


def gather_winner_masks(best_key, idx_bits: int, index_base: int, r_mask, s_mask, group=None):
    """Winners' R / S masks on every rank: after global_best, the rank owning
    budget b's winner (global index in [index_base, index_base + local count)) copies its
    rows into slot b of a zero [n_budget][2][n][W] int64 buffer; an all-reduce SUM (one
    contributor per slot) leaves every rank with all winners' masks, e.g. for cm_emit_plan.
    r_mask / s_mask: this rank's [local candidates][n][W] int64 tensors (round_and_evaluate
    with masks=True).  Slots of budgets with no feasible candidate stay zero."""
    import torch
    import torch.distributed as dist
    nb = best_key.numel()
    n, W = r_mask.shape[1], r_mask.shape[2]
    out = torch.zeros((nb, 2, n, W), dtype=torch.int64, device=r_mask.device)
    for b, k in enumerate(best_key.tolist()):
        if k == (1 << 63) - 1:
            continue
        idx = k & ((1 << idx_bits) - 1) if idx_bits else 0
        local = idx - index_base
        if 0 <= local < r_mask.shape[0]:
            out[b, 0] = r_mask[local]
            out[b, 1] = s_mask[local]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        with torch.cuda.nvtx.range("cm_gather_winner_masks"):
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def decode_keys(best_key, idx_bits: int):
    """Host decode of a key vector -> list of (cost, idx); (-1, -1) for 'none feasible'."""
    out = []
    for k in best_key.tolist():
        if k == (1 << 63) - 1:
            out.append((-1, -1))
        else:
            out.append((k >> idx_bits, k & ((1 << idx_bits) - 1) if idx_bits else 0))
    return out


# ----------------------------------------------------------------------------- NVLS keys
# The a8 MIN inside the reduce step: a multicast buffer spans the ranks' GPUs;
# every call reduces its keys with multimem.red.min into it (cm_eval_args.best_key_mc), and
# after all ranks' calls (one barrier) every GPU's replica holds the global per-budget keys --
# no all-reduce per step.

def share_fd(fd, group=None):
    """Give rank 0's file descriptor to every rank of the group (a duplicate on each rank;
    rank 0 gets its own fd back).  Over an abstract Unix socket whose name rank 0 broadcasts
    (SCM_RIGHTS); the process group only carries the name.  Host logic: no GPU involved."""
    import os
    import socket
    import uuid
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return fd
    name = [None]
    if rank == 0:
        name[0] = "\0cm_mc_" + uuid.uuid4().hex
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name[0])
        srv.listen(world)
    dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if rank == 0:
        for _ in range(world - 1):
            conn, _ = srv.accept()
            with conn:
                socket.send_fds(conn, [b"x"], [fd])
        srv.close()
        dist.barrier(group=group)
        return fd
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(name[0])
    with cli:
        _, fds, _, _ = socket.recv_fds(cli, 1, 1)
    dist.barrier(group=group)
    return fds[0] if fds else os.dup(fd)


class _CAI:
    """__cuda_array_interface__ view of raw device memory (no ownership)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3}


class MulticastKeys:
    """``n_keys`` int64 keys in an NVLink multicast buffer across the group's GPUs (cm_mc_*).

    .local  torch int64 tensor: this GPU's replica (pass as best_key; read after a barrier)
    .mc     int: the multicast address (pass as best_key_mc)
    Collective over the group (one process per GPU).  Raises CMError on every rank if any
    rank's stage fails (e.g. no multicast object on the box), instead of leaving the others
    waiting in the next collective."""

    def __init__(self, n_keys: int, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import CMError, _lib
        P = ctypes.c_void_p
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        rank = dist.get_rank(group) if world > 1 else 0
        src = (dist.get_global_rank(group, 0) if group is not None else 0) if world > 1 else 0
        self._lib = _lib
        self.handle = None
        h = P()

        def step(fn, where):
            """Run one stage on this rank; every rank learns whether all succeeded (a failed
            rank must not leave the others waiting in the next collective)."""
            err = ""
            try:
                st = fn()
                if st:
                    err = f"{where}: {_lib.cm_status_string(st).decode()}: {_lib.cm_mc_last_error().decode()}"
            except Exception as ex:  # pragma: no cover
                err = f"{where}: {ex!r}"
            errs = [err]
            if world > 1:
                errs = [None] * world
                dist.all_gather_object(errs, err, group=group)
            bad = [e for e in errs if e]
            if bad:
                self.close()
                raise CMError(5, "MulticastKeys: " + "; ".join(bad))

        nbytes = 8 * int(n_keys)
        fd = ctypes.c_int32(-1)
        step(lambda: (_lib.cm_mc_create(nbytes, world, ctypes.byref(h)) or
                      (world > 1 and _lib.cm_mc_export_fd(h, ctypes.byref(fd)))) if rank == 0 else 0,
             "cm_mc_create / export")
        self.handle = h if rank == 0 else None
        if world > 1:
            size = [int(_lib.cm_mc_size(h)) if rank == 0 else 0]
            dist.broadcast_object_list(size, src=src, group=group)
            got = share_fd(fd.value if rank == 0 else -1, group)
            step(lambda: _lib.cm_mc_import_fd(got, size[0], ctypes.byref(h)) if rank != 0 else 0, "cm_mc_import_fd")
            self.handle = h
        step(lambda: _lib.cm_mc_add_device(h), "cm_mc_add_device")   # all added before any binds
        uc, mc = P(), P()
        step(lambda: _lib.cm_mc_bind(h, ctypes.byref(uc), ctypes.byref(mc)), "cm_mc_bind")
        self.mc = int(mc.value)
        # a view of the replica: keep this object alive while the tensor is used
        self.local = torch.as_tensor(_CAI(int(uc.value), int(n_keys)), device="cuda")

    def reset(self):
        """Every replica to CM_KEY_NONE (each rank writes its own; barrier before the next
        call that reduces into it)."""
        self.local.fill_((1 << 63) - 1)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.cm_mc_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
