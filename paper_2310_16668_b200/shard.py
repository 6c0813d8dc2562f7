"""Multi-GPU apply: one process per GPU, whole level-1 subtrees per rank.

Every rank builds a sharded plan from the same full descriptor
(``sfmm_gpu_plan_create_sharded``).  An apply is

    begin   gather + upward pass of the owned subtrees, pack the ghost boxes
            (q and qhat) other ranks read;
    exchange  all-to-all of the packed ghosts (NCCL over NVLink via
            torch.distributed, on a side stream);
    mid     unpack, the translation tasks (one launch), pack the column sums
            of the cross-rank colleague pairs this rank evaluated for the
            other side;
    exchange  all-to-all of those column sums (second, smaller exchange);
    fin     add the staged and received column sums, downward pass, scatter of
            the owned points.
A colleague pair split across two ranks is evaluated once, by one of its two
owners (chosen to balance the ranks' work, plan_build.cpp); with
SFMM_SHARD_XSYM=0 both sides evaluate it and the second exchange disappears
(``end`` = mid + fin).  With
SFMM_SHARD_OVERLAP=1, begin also starts the tasks that read no ghost box so
they overlap the first exchange; measured slower, see DESIGN.md 6.

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
    counts = np.zeros(4 * n_ranks + 4, dtype=np.int64)
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
            "owned_points": owned[:n_owned],
            "send2_counts": counts[2 * n_ranks + 3:3 * n_ranks + 3].copy(),
            "recv2_counts": counts[3 * n_ranks + 3:4 * n_ranks + 3].copy(),
            "cut_level": int(counts[4 * n_ranks + 3])}


def T_runs(desc, n_ranks: int, rank: int):
    """Runs (src, len) of desc's T entries that `rank` owns, in the order of
    its compact operator blob, and their total (host-only)."""
    lib = _abi.gpu_lib()
    st = _struct(desc)
    nr, ne = C.c_int64(), C.c_int64()
    _raise(lib.sfmm_gpu_shard_T_runs(C.byref(st), n_ranks, rank, C.byref(nr), None, C.byref(ne)))
    runs = np.zeros((max(1, nr.value), 2), dtype=np.int64)
    _raise(lib.sfmm_gpu_shard_T_runs(C.byref(st), n_ranks, rank, C.byref(nr), runs.ctypes.data,
                                     C.byref(ne)))
    return runs[: nr.value], ne.value


def pack_T(src_ptr: int, runs: np.ndarray, scalars_per_entry: int, out, device: int,
           stream: int = 0) -> None:
    """Copies the runs of a device-resident full T (src_ptr, e.g. the GPU
    skeletonizer's result) into the torch float64 device tensor `out`."""
    runs = np.ascontiguousarray(runs, dtype=np.int64)
    _raise(_abi.gpu_lib().sfmm_gpu_copy_runs(C.c_void_p(src_ptr), runs.ctypes.data, len(runs),
                                             scalars_per_entry, C.c_void_p(out.data_ptr()), device,
                                             C.c_void_p(stream or None)))


class ShardedPlan:
    """This rank's part of a sharded plan (device resident).  T_owned: the
    rank's operator blob on its device (pack_T / T_runs), for descriptors
    shared without T."""

    def __init__(self, desc, n_ranks: int, rank: int, device: int = 0, T_owned=None):
        lib = _abi.gpu_lib()
        st = _struct(desc)
        self._h = None
        h = C.c_void_p()
        if T_owned is not None and getattr(T_owned, "owner", None) is not None:
            _raise(lib.sfmm_gpu_plan_create_sharded_owned(
                C.byref(st), C.c_void_p(T_owned.data_ptr()), device, n_ranks, rank,
                T_owned.owner.ctypes.data, C.byref(h)))
        elif T_owned is not None:
            _raise(lib.sfmm_gpu_plan_create_sharded_T(C.byref(st), C.c_void_p(T_owned.data_ptr()),
                                                      device, n_ranks, rank, C.byref(h)))
        else:
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
        send2 = np.zeros(n_ranks, dtype=np.int64)
        recv2 = np.zeros(n_ranks, dtype=np.int64)
        cut = C.c_int(1)
        self.cross_symmetric = bool(lib.sfmm_gpu_shard_info2(self._h, send2.ctypes.data,
                                                              recv2.ctypes.data, C.byref(cut)))
        self.cut_level = cut.value  # 1: level-1 subtrees per rank, 2: level-2 (level 1 shared)
        self.send2_counts = send2 * self.sw  # in doubles
        self.recv2_counts = recv2 * self.sw
        self._bufs = None
        self._bufs2 = None

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

    def buffers2(self):
        """Device send / receive buffers of the second exchange."""
        import torch
        if self._bufs2 is None:
            dev = f"cuda:{self.device}"
            self._bufs2 = (torch.empty(max(1, int(self.send2_counts.sum())), dtype=torch.float64, device=dev),
                           torch.empty(max(1, int(self.recv2_counts.sum())), dtype=torch.float64, device=dev))
        return self._bufs2

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

    def mid(self, stream: int, packed_event: int = 0) -> None:
        _, recv = self.buffers()
        send2, _ = self.buffers2()
        _raise(_abi.gpu_lib().sfmm_gpu_apply_mid(self._h, C.c_void_p(recv.data_ptr()),
                                                 C.c_void_p(send2.data_ptr()),
                                                 C.c_void_p(stream or None),
                                                 C.c_void_p(packed_event or None)))

    def fin(self, q_dev, u_dev, stream: int) -> None:
        _, recv2 = self.buffers2()
        _raise(_abi.gpu_lib().sfmm_gpu_apply_fin(self._h, C.c_void_p(q_dev.data_ptr()),
                                                 C.c_void_p(recv2.data_ptr()),
                                                 C.c_void_p(u_dev.data_ptr()),
                                                 C.c_void_p(stream or None)))

    # ---- exchange inside the library (NCCL, one process per GPU) ----------
    def attach_nccl(self, unique_id: bytes) -> None:
        """Joins this rank to the NCCL communicator of id `unique_id` (from
        nccl_unique_id() on rank 0, broadcast by the caller); sfmm_gpu_apply /
        apply() on this plan are then collective, both exchanges run inside the
        library (sfmm_gpu_plan_attach_nccl)."""
        _set_nccl_path()
        buf = C.create_string_buffer(bytes(unique_id), NCCL_ID_BYTES)
        _raise(_abi.gpu_lib().sfmm_gpu_plan_attach_nccl(self._h, buf, self.n_ranks, self.rank))

    def set_output(self, owned_only: bool) -> None:
        """Collective applies write the whole u on every rank (default, one
        in-place all-reduce) or only this rank's owned points."""
        _raise(_abi.gpu_lib().sfmm_gpu_set_output(
            self._h, _abi.SFMM_OUTPUT_OWNED if owned_only else _abi.SFMM_OUTPUT_FULL))

    def apply(self, q_dev, u_dev, stream: int) -> None:
        """One collective apply (NCCL-attached plan) enqueued on `stream`."""
        _raise(_abi.gpu_lib().sfmm_gpu_apply_async(self._h, C.c_void_p(q_dev.data_ptr()),
                                                   C.c_void_p(u_dev.data_ptr()), 1,
                                                   C.c_void_p(stream or None)))

    def apply_host(self, q: np.ndarray, out: np.ndarray) -> None:
        """Collective apply through the public host-buffer entry point."""
        _raise(_abi.gpu_lib().sfmm_gpu_apply(self._h, q.ctypes.data, out.ctypes.data, 1,
                                             _abi.SFMM_HOST_BUFFERS, None))

    def close(self) -> None:
        if self._h is not None:
            _abi.gpu_lib().sfmm_gpu_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


NCCL_ID_BYTES = 128


def _set_nccl_path() -> None:
    """Points the library's run-time NCCL load at the NCCL torch ships (the
    one torch.distributed already uses in this process), unless set."""
    import os
    if os.environ.get("SFMM_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        base = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(base):
            os.environ["SFMM_NCCL_LIB"] = base
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL communicator id (rank 0), 128 bytes."""
    _set_nccl_path()
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _raise(_abi.gpu_lib().sfmm_gpu_nccl_unique_id(buf))
    return buf.raw


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


def _all_to_all(stream, comm_stream, ready, send, recv, send_counts, recv_counts, n_ranks):
    """recv <- all-to-all(send) on comm_stream after `ready`; stream waits for it."""
    import torch
    import torch.distributed as dist
    done = torch.cuda.Event()
    with torch.cuda.stream(comm_stream):
        comm_stream.wait_event(ready)
        if n_ranks > 1:
            dist.all_to_all_single(recv[: int(recv_counts.sum())], send[: int(send_counts.sum())],
                                   output_split_sizes=[int(x) for x in recv_counts],
                                   input_split_sizes=[int(x) for x in send_counts])
        done.record(comm_stream)
    stream.wait_event(done)


def apply_distributed(plan: ShardedPlan, q_dev, u_dev, stream=None, comm_stream=None) -> None:
    """One sharded apply with the all-to-alls on torch.distributed (NCCL) on a
    side stream: ghosts after the upward pass, then (cross-symmetric plans)
    the column sums after the translations.  u_dev receives the owned points
    (other entries untouched)."""
    import torch
    stream, fence = _work_stream(stream, plan.device)
    comm_stream = comm_stream or torch.cuda.Stream(plan.device)
    packed = torch.cuda.Event()
    packed.record(stream)  # materialise the event; begin() re-records it after packing
    send, recv = plan.buffers()
    plan.begin(q_dev, stream.cuda_stream, packed.cuda_event)
    _all_to_all(stream, comm_stream, packed, send, recv, plan.send_counts, plan.recv_counts,
                plan.n_ranks)
    if plan.cross_symmetric:
        packed2 = torch.cuda.Event()
        packed2.record(stream)
        send2, recv2 = plan.buffers2()
        plan.mid(stream.cuda_stream, packed2.cuda_event)
        _all_to_all(stream, comm_stream, packed2, send2, recv2, plan.send2_counts,
                    plan.recv2_counts, plan.n_ranks)
        plan.fin(q_dev, u_dev, stream.cuda_stream)
    else:
        plan.end(q_dev, u_dev, stream.cuda_stream)
    fence()


def _copy_exchange(plans, send_counts, recv_counts, bufs):
    n = len(plans)
    send_off = [np.concatenate([[0], np.cumsum(send_counts(p))]) for p in plans]
    recv_off = [np.concatenate([[0], np.cumsum(recv_counts(p))]) for p in plans]
    for src in range(n):
        for dst in range(n):
            cnt = int(send_counts(plans[src])[dst])
            assert cnt == int(recv_counts(plans[dst])[src])
            if cnt == 0:
                continue
            s0, d0 = int(send_off[src][dst]), int(recv_off[dst][src])
            bufs(plans[dst])[1][d0:d0 + cnt].copy_(bufs(plans[src])[0][s0:s0 + cnt])


def apply_virtual(plans: list[ShardedPlan], q_dev, u_dev, stream=None) -> None:
    """All ranks' shards on ONE GPU, run one after another (no kernel waits on
    another rank); the all-to-alls become device-to-device copies.  Used to
    test the sharded path where only one GPU is available."""
    import torch
    stream, fence = _work_stream(stream, plans[0].device)
    for p in plans:
        p.begin(q_dev, stream.cuda_stream, 0)
    with torch.cuda.stream(stream):
        _copy_exchange(plans, lambda p: p.send_counts, lambda p: p.recv_counts,
                       lambda p: p.buffers())
    if plans[0].cross_symmetric:
        for p in plans:
            p.mid(stream.cuda_stream)
        with torch.cuda.stream(stream):
            _copy_exchange(plans, lambda p: p.send2_counts, lambda p: p.recv2_counts,
                           lambda p: p.buffers2())
        for p in plans:
            p.fin(q_dev, u_dev, stream.cuda_stream)
    else:
        for p in plans:
            p.end(q_dev, u_dev, stream.cuda_stream)
    fence()


# ---------------------------------------------------------------------------
# distributed precompute (no rank holds every operator)
# ---------------------------------------------------------------------------

def subtree_owners(hp, n_ranks: int) -> np.ndarray:
    """Rank of every box from the tree alone (sfmm_gpu_subtree_owners):
    Morton-contiguous ranges of level-1 subtrees; -1 above level 1."""
    a = hp.tree_arrays()
    owner = np.zeros(int(a.n_boxes), dtype=np.int32)
    _raise(_abi.gpu_lib().sfmm_gpu_subtree_owners(C.byref(a), n_ranks, owner.ctypes.data))
    return owner


_IDX = ("iv", "skel_pos", "red_pos")
_OFF = {"iv": "iv_off", "skel_pos": "sk_off", "red_pos": "rd_off"}


def local_index_data(hp, owner: np.ndarray, rank: int) -> dict:
    """This rank's share of the skeleton index data: for each box it owns
    (ascending id) the index_vec / skel_pos / red_pos segment lengths and
    contents and its parent_offset.  The subset build leaves every other box
    empty, so the packed arrays are the local arrays themselves."""
    d = hp.descriptor().arrays
    boxes = np.nonzero(owner == rank)[0].astype(np.int32)
    out = {"boxes": boxes, "poff": np.asarray(d["box_parent_offset"])[boxes].copy()}
    for f in _IDX:
        off = np.asarray(d[_OFF[f]])
        out["len_" + f] = np.diff(off)[boxes].astype(np.int64)
        out[f] = np.asarray(d[f]).copy()
        assert out[f].size == int(out["len_" + f].sum()), "subset result holds unowned boxes"
    return out


def _place(dst: np.ndarray, dst_off: np.ndarray, boxes: np.ndarray, lens: np.ndarray,
           src: np.ndarray) -> None:
    if src.size == 0:
        return
    starts = dst_off[boxes]
    first = np.concatenate([[0], np.cumsum(lens)[:-1]])
    dst[np.repeat(starts - first, lens) + np.arange(src.size)] = src


def assemble_descriptor(hp, parts: list) -> PlanDescriptor:
    """The full plan descriptor (no T) from every rank's index data and this
    rank's tree: what a single skeletonization of the whole tree gives, box
    for box (each box's skeleton depends only on its own subtree)."""
    base = hp.descriptor()
    arrays = dict(base.arrays)
    scalars = dict(base.scalars)
    nb = int(scalars["n_boxes"])
    level = np.asarray(arrays["box_level"])
    lens = {f: np.zeros(nb, dtype=np.int64) for f in _IDX}
    poff = np.zeros(nb, dtype=np.int32)
    for p in parts:
        for f in _IDX:
            lens[f][p["boxes"]] = p["len_" + f]
        poff[p["boxes"]] = p["poff"]
    for f in _IDX:
        off = np.concatenate([[0], np.cumsum(lens[f])]).astype(np.int64)
        arrays[_OFF[f]] = off
        dst = np.zeros(int(off[-1]), dtype=np.int32)
        for p in parts:
            _place(dst, off, p["boxes"], p["len_" + f], p[f])
        arrays[f] = dst
    n, k = lens["iv"], lens["skel_pos"]
    arrays["T_off"] = np.concatenate([[0], np.cumsum(np.where(level >= 2, k * (n - k), 0))]).astype(np.int64)
    arrays["box_parent_offset"] = poff
    arrays["T"] = np.zeros(0, dtype=np.float64)
    return PlanDescriptor(scalars, arrays)


def distributed_precompute(kernel: int, pts: np.ndarray, leaf_cap: int, tol: float,
                           kappa: float, n_ranks: int, rank: int, device: int, all_gather):
    """One rank's share of the precompute: the tree (every rank builds the
    same one), the tree-only ownership, the skeletons of this rank's level-1
    subtrees only (operators stay on `device`), then the index data of all
    ranks via all_gather(part) -> [part of rank 0, 1, ...] to form the full
    descriptor.  Returns (descriptor without T, host plan holding this rank's
    operators, owner)."""
    from . import host
    hp = host.HostPlan.build_tree_gpu(pts, leaf_cap, device)
    owner = subtree_owners(hp, n_ranks)
    hp.skeletonize(kernel, tol, kappa, device=device, host_T=False, box_mask=owner == rank)
    parts = all_gather(local_index_data(hp, owner, rank))
    return assemble_descriptor(hp, parts), hp, owner


class OwnedShardedPlan(ShardedPlan):
    """A rank plan of the distributed precompute: the ownership it was
    skeletonized for, its operators taken from the subset build's device T
    (sfmm_gpu_plan_create_sharded_owned)."""

    def __init__(self, desc, n_ranks: int, rank: int, device: int, T_ptr: int, owner: np.ndarray):
        self._owner = np.ascontiguousarray(owner, dtype=np.int32)
        super().__init__(desc, n_ranks, rank, device, T_owned=_OwnedT(T_ptr, self._owner))


class _OwnedT:
    """T_owned for ShardedPlan: a raw device pointer plus the ownership."""

    def __init__(self, ptr: int, owner: np.ndarray):
        self.ptr, self.owner = ptr, owner

    def data_ptr(self) -> int:
        return self.ptr
