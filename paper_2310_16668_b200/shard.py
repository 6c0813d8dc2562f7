"""Multi-GPU apply: one process per GPU, whole level-1 subtrees per rank.

Every rank builds a sharded plan from the same full descriptor
(``sfmm_gpu_plan_create_sharded``).  An apply is

    begin   gather + upward pass of the owned subtrees, pack the ghost boxes
            (q and qhat) other ranks read;
    exchange  all-to-all of the packed ghosts (NCCL over NVLink via
            torch.distributed, on a side stream);
    end     unpack, the translation tasks (one launch), staged column sums,
            downward pass, scatter of the owned points.
(With SFMM_SHARD_OVERLAP=1, begin also starts the tasks that read no ghost box
so they overlap the exchange; measured slower.)

The reference is single-process (SPEC.md non-goal "distributed trees"); this is
the B200-native extension described in SURVEY.md 8(e) and DESIGN.md 6.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import PlanDesc, PlanDescriptor
from .api import _raise


def _struct(desc) -> PlanDesc:
    if isinstance(desc, PlanDescriptor):
        return desc.struct
    if isinstance(desc, PlanDesc):
        return desc
    raise TypeError("expected a PlanDescriptor or a PlanDesc")


def describe(desc, n_ranks: int, rank: int) -> dict:
    """Host-only shard layout of `rank` (no GPU needed)."""
    lib = _abi.gpu_lib()
    st = _struct(desc)
    counts = np.zeros(2 * n_ranks + 3, dtype=np.int64)
    _raise(lib.sfmm_gpu_shard_describe(C.byref(st), n_ranks, rank, counts.ctypes.data, None, None,
                                       None, None))
    send = counts[:n_ranks].copy()
    recv = counts[n_ranks:2 * n_ranks].copy()
    n_owned = int(counts[2 * n_ranks])
    owner = np.zeros(int(st.n_boxes), dtype=np.int32)
    pack = np.zeros(max(1, int(send.sum())), dtype=np.int64)
    unpack = np.zeros(max(1, int(recv.sum())), dtype=np.int64)
    owned = np.zeros(max(1, n_owned), dtype=np.int32)
    _raise(lib.sfmm_gpu_shard_describe(C.byref(st), n_ranks, rank, counts.ctypes.data,
                                       owner.ctypes.data, pack.ctypes.data, unpack.ctypes.data,
                                       owned.ctypes.data))
    return {"send_counts": send, "recv_counts": recv, "n_owned_points": n_owned,
            "n_ghost_boxes": int(counts[2 * n_ranks + 1]), "n_owned_boxes": int(counts[2 * n_ranks + 2]),
            "owner": owner, "pack_idx": pack[: int(send.sum())], "unpack_idx": unpack[: int(recv.sum())],
            "owned_points": owned[:n_owned]}


class ShardedPlan:
    """This rank's part of a sharded plan (device resident)."""

    def __init__(self, desc, n_ranks: int, rank: int, device: int = 0):
        lib = _abi.gpu_lib()
        st = _struct(desc)
        self._h = None
        h = C.c_void_p()
        _raise(lib.sfmm_gpu_plan_create_sharded(C.byref(st), device, n_ranks, rank, C.byref(h)))
        self._h = h
        self.n_ranks, self.rank, self.device = n_ranks, rank, device
        self.n_points = int(st.n_points)
        self.is_complex = int(st.kernel) in (_abi.HELMHOLTZ2D, _abi.HELMHOLTZ3D)
        self.sw = 2 if self.is_complex else 1  # doubles per scalar
        send = np.zeros(n_ranks, dtype=np.int64)
        recv = np.zeros(n_ranks, dtype=np.int64)
        owned = C.c_int64(0)
        ghosts = C.c_int64(0)
        _raise(lib.sfmm_gpu_shard_info(self._h, send.ctypes.data, recv.ctypes.data,
                                       C.byref(owned), C.byref(ghosts)))
        self.send_counts = send * self.sw  # in doubles
        self.recv_counts = recv * self.sw
        self.n_owned_points = owned.value
        self.n_ghost_boxes = ghosts.value
        self._bufs = None

    def info(self) -> _abi.PlanInfo:
        """sfmm_gpu_plan_info_get of this rank's plan (pair counts are global)."""
        from .api import _raise
        inf = _abi.PlanInfo()
        _raise(_abi.gpu_lib().sfmm_gpu_plan_info_get(self._h, C.byref(inf)))
        return inf

    def buffers(self):
        """Device send / receive buffers (torch float64), allocated once."""
        import torch
        if self._bufs is None:
            dev = f"cuda:{self.device}"
            self._bufs = (torch.empty(max(1, int(self.send_counts.sum())), dtype=torch.float64, device=dev),
                          torch.empty(max(1, int(self.recv_counts.sum())), dtype=torch.float64, device=dev))
        return self._bufs

    def begin(self, q_dev, stream: int, packed_event: int = 0) -> None:
        send, _ = self.buffers()
        _raise(_abi.gpu_lib().sfmm_gpu_apply_begin(self._h, C.c_void_p(q_dev.data_ptr()),
                                                   C.c_void_p(send.data_ptr()),
                                                   C.c_void_p(stream or None),
                                                   C.c_void_p(packed_event or None)))

    def end(self, q_dev, u_dev, stream: int) -> None:
        _, recv = self.buffers()
        _raise(_abi.gpu_lib().sfmm_gpu_apply_end(self._h, C.c_void_p(q_dev.data_ptr()),
                                                 C.c_void_p(recv.data_ptr()),
                                                 C.c_void_p(u_dev.data_ptr()),
                                                 C.c_void_p(stream or None)))

    def close(self) -> None:
        if self._h is not None:
            _abi.gpu_lib().sfmm_gpu_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _work_stream(stream, device):
    """The C ABI reads a NULL stream as the plan's own stream, so work that must
    be ordered with torch's legacy default stream runs on a side stream that is
    fenced against it (returns the stream and a closing fence)."""
    import torch
    cur = stream or torch.cuda.current_stream(device)
    if cur.cuda_stream != 0:
        return cur, lambda: None
    side = torch.cuda.Stream(device)
    side.wait_stream(cur)
    return side, lambda: cur.wait_stream(side)


def apply_distributed(plan: ShardedPlan, q_dev, u_dev, stream=None, comm_stream=None) -> None:
    """One sharded apply with the ghost all-to-all on torch.distributed (NCCL),
    after the upward pass (overlapping the interior tasks with SFMM_SHARD_OVERLAP=1).  u_dev receives the owned
    points (other entries untouched)."""
    import torch
    import torch.distributed as dist
    stream, fence = _work_stream(stream, plan.device)
    comm_stream = comm_stream or torch.cuda.Stream(plan.device)
    packed = torch.cuda.Event()
    done = torch.cuda.Event()
    packed.record(stream)  # materialise the event; begin() re-records it after packing
    send, recv = plan.buffers()
    # begin records `packed` on `stream` right after the pack kernel
    plan.begin(q_dev, stream.cuda_stream, packed.cuda_event)
    with torch.cuda.stream(comm_stream):
        comm_stream.wait_event(packed)
        if plan.n_ranks > 1:
            dist.all_to_all_single(recv[: int(plan.recv_counts.sum())],
                                   send[: int(plan.send_counts.sum())],
                                   output_split_sizes=[int(x) for x in plan.recv_counts],
                                   input_split_sizes=[int(x) for x in plan.send_counts])
        done.record(comm_stream)
    stream.wait_event(done)
    plan.end(q_dev, u_dev, stream.cuda_stream)
    fence()


def apply_virtual(plans: list[ShardedPlan], q_dev, u_dev, stream=None) -> None:
    """All ranks' shards on ONE GPU, run one after another (no kernel waits on
    another rank); the all-to-all becomes device-to-device copies.  Used to
    test the sharded path where only one GPU is available."""
    import torch
    stream, fence = _work_stream(stream, plans[0].device)
    for p in plans:
        p.begin(q_dev, stream.cuda_stream, 0)
    n = len(plans)
    send_off = [np.concatenate([[0], np.cumsum(p.send_counts)]) for p in plans]
    recv_off = [np.concatenate([[0], np.cumsum(p.recv_counts)]) for p in plans]
    with torch.cuda.stream(stream):
        for src in range(n):
            for dst in range(n):
                cnt = int(plans[src].send_counts[dst])
                assert cnt == int(plans[dst].recv_counts[src])
                if cnt == 0:
                    continue
                s0, d0 = int(send_off[src][dst]), int(recv_off[dst][src])
                plans[dst].buffers()[1][d0:d0 + cnt].copy_(plans[src].buffers()[0][s0:s0 + cnt])
    for p in plans:
        p.end(q_dev, u_dev, stream.cuda_stream)
    fence()
