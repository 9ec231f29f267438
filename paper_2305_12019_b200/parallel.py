"""Sample-sharded solves across GPUs.

Z~ is split by contiguous blocks of sample columns; each rank (one process per
GPU) uploads its block and its slices of y, e and the weights.  Feature-space
work (w, u, rho, h, the DIRECT factor, PSQMR vectors) is replicated and stays
bit-identical across ranks; every sum over samples is all-reduced -- the
d-partial of each Z~ t together with the n-sums of the same pass (one bundle
per reduction point), the n-sums of the per-sample passes, and once at setup
Z~y, ||Z~||_F^2, the Jacobi diagonal and (DIRECT) the d x d Gram.

Communicators:
  * ``NcclCommunicator``: NCCL over NVLink/NVSwitch, bootstrapped with a
    ``torch.distributed`` broadcast of the NCCL unique id (torchrun launches).
  * ``HostCommunicator``: all-reduce through a host callback (gloo process
    groups, or threads emulating ranks on one GPU in tests).

``solve_on_devices`` (also ``sgs_admm_solve(..., devices=[...])``) drives all
ranks from one process, one host thread per GPU.

SMW2 couples all samples through its n x n Gram, so it is not sharded
(``bench.py --gpus N`` runs replicas for config 2).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Callable, Optional

import numpy as np

from . import _lib
from .solver import DeviceProblem, ProblemData, _check, device_problem
from .sparse import SparseMatrixCSC


def shard_bounds(n: int, nranks: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced sample block [lo, hi) of `rank`."""
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    return n * rank // nranks, n * (rank + 1) // nranks


def shard_problem(data: ProblemData, rank: int, nranks: int) -> ProblemData:
    """The local ProblemData of `rank`: its block of Z~ columns and the
    matching slices of y, e and the weights (z_scale, C, q unchanged)."""
    lo, hi = shard_bounds(data.n, nranks, rank)
    z = data.z_tilde
    if z.is_dense:
        zl = SparseMatrixCSC.from_dense_samples(z.dense_samples()[lo:hi])
    else:
        cp = z.colptr
        a, b = int(cp[lo]), int(cp[hi])
        zl = SparseMatrixCSC(z.nrows, hi - lo, cp[lo:hi + 1] - a, z.rowidx[a:b], z.values[a:b])
    return ProblemData(zl, data.y[lo:hi], data.e[lo:hi], data.weights[lo:hi], data.C, data.q, data.z_scale)


class HostCommunicator:
    """Sum-all-reduce through a Python function ``allreduce(np.ndarray) ->
    np.ndarray`` (e.g. torch.distributed with gloo, or a thread barrier)."""

    def __init__(self, allreduce: Callable[[np.ndarray], np.ndarray], nranks: int, rank: int):
        self.allreduce, self.nranks, self.rank = allreduce, nranks, rank
        self._err: list = []

        def _cb(user, buf, count):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(count,))
                arr[:] = self.allreduce(arr.copy())
                return 0
            except BaseException as exc:  # pragma: no cover - surfaced by the caller
                self._err.append(exc)
                return 1

        self._cfun = _lib.ALLREDUCE_CB(_cb)

    def attach(self, dp: DeviceProblem, n_global: int) -> None:
        lib = _lib.load()
        _check(lib.gdwd_comm_init_host(dp.ctx, self.nranks, self.rank, self._cfun, None, int(n_global)), dp.ctx,
               "comm_init_host")
        dp.comm = self
        dp.n_global = int(n_global)


def pin_nccl_determinism() -> None:
    """Fix NCCL's algorithm and protocol (ring, simple) unless the user chose
    them: the fp64 sum of an all-reduce is then formed in the same order on
    every run, so sharded solves are bitwise reproducible run to run (NVLS /
    tree selection can otherwise change with message size or topology).
    Must run before the first NCCL communicator of the process (NCCL reads
    these once); bench.py calls it before torch.distributed's own init."""
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")


class NcclCommunicator:
    """NCCL communicator over the ranks of a torch.distributed group."""

    def __init__(self, nranks: int, rank: int, broadcast_id: Callable[[Optional[bytes]], bytes]):
        """``broadcast_id(id_or_None)``: rank 0 passes its id, every rank gets it back."""
        pin_nccl_determinism()
        try:  # torch's bundled libnccl.so.2 first: the library's dlopen then binds the same one
            import torch  # noqa: F401
        except ImportError:
            pass
        lib = _lib.load()
        uid = None
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            _check(lib.gdwd_comm_unique_id(buf), None, "nccl unique id")
            uid = bytes(buf)
        self.uid = broadcast_id(uid)
        self.nranks, self.rank = nranks, rank

    @classmethod
    def from_torch(cls) -> "NcclCommunicator":
        import torch.distributed as dist

        def bcast(uid):
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            return obj[0]

        return cls(dist.get_world_size(), dist.get_rank(), bcast)

    def attach(self, dp: DeviceProblem, n_global: int) -> None:
        lib = _lib.load()
        ida = (C.c_uint8 * 128).from_buffer_copy(self.uid)
        _check(lib.gdwd_comm_init_nccl(dp.ctx, self.nranks, self.rank, ida, int(n_global)), dp.ctx,
               "comm_init_nccl")
        dp.comm = self
        dp.n_global = int(n_global)


def attach(local: ProblemData, comm, n_global: int, device: Optional[int] = None) -> DeviceProblem:
    """Upload the local shard (if not yet resident) and join the communicator;
    later ``sgs_admm_solve(local, ...)`` calls run sharded."""
    # hint ITERATIVE: a shard needs nothing factored during its upload (the
    # Grams a sharded solve uses are summed over the shards at setup)
    dp = device_problem(local, device, (_lib.BACKEND_CODE["iterative"], 1.0))
    comm.attach(dp, n_global)
    return dp


def global_train_error(result, local: ProblemData, allreduce: Callable[[np.ndarray], np.ndarray],
                       n_global: int) -> float:
    """Train error over all shards (solver.py:558-559): each rank counts its
    misclassified samples from its slice of y and Z~^T w."""
    st = result.final_state
    ztw = result.extras_ztw if hasattr(result, "extras_ztw") else None
    if ztw is None:
        ztw = device_problem(local).state()["ztw"]
    scores = st.beta + local.y * ztw
    bad = np.array([float(np.sum(local.y * np.sign(scores) <= 0.0))])
    return 100.0 * float(allreduce(bad)[0]) / n_global


def solve_on_devices(data: ProblemData, config, devices, comm: str = "nccl", **kw):
    """``sgs_admm_solve`` sharded over several GPUs from ONE process (SURVEY.md
    section 5: one host thread per device, NCCL over NVLink between them), so a
    multi-GPU solve is still a plain call -- no torchrun.

    ``data`` is the global problem; rank r gets the r-th contiguous block of
    samples and drives ``devices[r]``.  ``comm="host"`` exchanges through a
    host all-reduce instead (``ThreadRanks``; lets several ranks share one GPU
    in tests, their kernels never waiting on one another).  Returns rank 0's
    SolveResult with the sample-space iterates (r, xi, alpha) of all ranks
    concatenated; feature-space state is replicated and bit-identical."""
    from .solver import as_problem, sgs_admm_solve

    data = as_problem(data)
    devices = [int(x) for x in devices]
    world = len(devices)
    if world < 1:
        raise ValueError("need at least one device")
    if kw.get("callback") is not None:
        raise NotImplementedError("per-iteration callbacks need the global iterate; use devices=None")
    if comm not in ("nccl", "host"):
        raise ValueError("comm must be 'nccl' or 'host'")
    n = data.n
    locals_ = [shard_problem(data, r, world) for r in range(world)]
    for r in range(world):  # uploads in rank order (host memory bandwidth is shared anyway)
        device_problem(locals_[r], devices[r])
    ranks = ThreadRanks(world)
    if comm == "nccl":
        lib = _lib.load()
        buf = (C.c_uint8 * 128)()
        _check(lib.gdwd_comm_unique_id(buf), None, "nccl unique id")
        uid = bytes(buf)
    outs: list = [None] * world
    errs: list = []

    def run(r: int) -> None:
        try:
            if comm == "nccl":
                cm = NcclCommunicator(world, r, lambda _id: uid)
            else:
                cm = HostCommunicator(ranks.allreduce_for(r), world, r)
            attach(locals_[r], cm, n, devices[r])
            outs[r] = sgs_admm_solve(locals_[r], config, device=devices[r], **kw)
        except BaseException as exc:
            errs.append(exc)
            ranks.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,), name=f"gdwd-rank{r}") for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    real = [e for e in errs if not isinstance(e, threading.BrokenBarrierError)]
    if errs:
        raise (real or errs)[0]
    out = outs[0]
    st = out.final_state
    for key in ("r", "xi", "alpha"):
        setattr(st, key, np.concatenate([getattr(o.final_state, key) for o in outs]))
    return out


class ThreadRanks:
    """Emulate `nranks` ranks as threads of one process (sum all-reduce via a
    barrier) -- the host side of virtual-rank tests on a single GPU."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots: list = [None] * nranks
        self.result = None

    def allreduce_for(self, rank: int) -> Callable[[np.ndarray], np.ndarray]:
        def ar(x: np.ndarray) -> np.ndarray:
            self.slots[rank] = x
            if self.barrier.wait() == 0:
                acc = self.slots[0].copy()
                for r in range(1, self.nranks):
                    acc += self.slots[r]  # fixed rank order: identical on every rank
                self.result = acc
            self.barrier.wait()
            out = self.result.copy()
            self.barrier.wait()
            return out

        return ar


__all__ = ["HostCommunicator", "NcclCommunicator", "ThreadRanks", "attach", "global_train_error",
           "shard_bounds", "shard_problem", "solve_on_devices"]
