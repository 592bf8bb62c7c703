"""Thin Python binding of the qsim_* C-ABI (argument marshalling only).

PyTorch supplies device memory (the shards), the CUDA stream and, for
multi-GPU runs, the process group used to broadcast the NCCL unique id.
Every step of the gate path runs in libqsim_b200.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _native as N

G_1Q, G_CTRL, G_PERM, G_SWAP = 0, 1, 2, 3


def torch_float64():
    import torch
    return torch.float64


class QsimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        name = N.STATUS[status] if 0 <= status < len(N.STATUS) else str(status)
        super().__init__(f"{name}: {msg}")
        self.status = status
        self.name = name


def _u4(u) -> "ctypes.Array":
    arr = (N.c128 * 4)()
    for k in range(4):
        z = complex(u[k])
        arr[k].re, arr[k].im = z.real, z.imag
    return arr


def pack_gates(gates: Sequence) -> tuple:
    """Marshal gate records (objects with kind/target/controls/targets/u/perm,
    e.g. workloads.Gate) into a qsim_gate array.  Returns (array, keepalive)."""
    arr = (N.qsim_gate * max(1, len(gates)))()
    keep = []
    for i, g in enumerate(gates):
        r = arr[i]
        r.kind = g.kind
        if g.kind in (G_1Q, G_CTRL):
            r.target = g.target
            r.n_controls = len(g.controls)
            for j, c in enumerate(g.controls):
                r.controls[j] = c
            for k in range(4):
                z = complex(g.u[k])
                r.u[k].re, r.u[k].im = z.real, z.imag
        elif g.kind == G_PERM:
            r.n_controls = len(g.controls)
            for j, c in enumerate(g.controls):
                r.controls[j] = c
            r.n_targets = len(g.targets)
            for j, t in enumerate(g.targets):
                r.targets[j] = t
            p = np.ascontiguousarray(g.perm, dtype=np.uint32)
            keep.append(p)
            r.perm = p.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        elif g.kind == G_SWAP:
            r.targets[0], r.targets[1] = g.targets[0], g.targets[1]
        else:
            raise ValueError(f"unknown gate kind {g.kind}")
    return arr, keep


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    s = N.lib().qsim_get_unique_id(buf)
    if s != 0:
        raise QsimError(s, "ncclGetUniqueId failed")
    return bytes(buf)


def probe_peaks(fp64: bool = True, copy: bool = True) -> dict:
    """Measured roofline denominators of the current CUDA device
    (qsim_probe_peaks): FP64 FMA-pipe TFLOP/s and streaming-copy GB/s."""
    f, b = ctypes.c_double(0), ctypes.c_double(0)
    s = N.lib().qsim_probe_peaks(ctypes.byref(f) if fp64 else None, ctypes.byref(b) if copy else None)
    if s != 0:
        raise QsimError(s, "qsim_probe_peaks")
    return {"fp64_tflops": f.value if fp64 else None, "copy_gbs": b.value if copy else None}


def get_loopback_id() -> bytes:
    """Id of a new loopback group (QSim(..., transport="loopback", nccl_id=id))."""
    buf = (ctypes.c_uint8 * 128)()
    s = N.lib().qsim_get_loopback_id(buf)
    if s != 0:
        raise QsimError(s, "qsim_get_loopback_id")
    return bytes(buf)


def run_loopback(n: int, n_ranks: int, body, **kw) -> list:
    """Run the SPMD program body(sim, rank) -> result on n_ranks loopback
    ranks: one QSim per rank, each driven by its own host thread (the ctypes
    calls release the GIL), all on the current device.  Returns the results
    in rank order; re-raises the first exception."""
    import threading
    cid = get_loopback_id()
    out, errs = [None] * n_ranks, [None] * n_ranks

    def worker(r):
        sim = None
        try:
            sim = QSim(n, n_ranks=n_ranks, transport="loopback", rank=r, nccl_id=cid, **kw)
            out[r] = body(sim, r)
        except BaseException as e:  # noqa: BLE001 (reported below)
            errs[r] = e
        finally:
            if sim is not None:
                sim.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(n_ranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out


GLOBAL_POLICY = {"remap": 0, "pairwise": 1, "auto": 2}


def plan_json(n: int, n_ranks: int, gates: Sequence, fusion: int = 1, policy: Optional[str] = None,
              block_fusion: bool = True, low_remap: bool = True, remap_lookahead: Optional[int] = None,
              key_check: bool = False, candidate: Optional[int] = None, overlap: bool = False,
              readout: bool = False) -> str:
    """Host-only planner introspection (no GPU needed).  fusion=2 also
    NVRTC-compiles the pass-specialised kernels (reported under "jit");
    key_check=True only generates their sources and checks that equal kernel-
    cache keys mean equal sources across every plan checked in this process;
    policy: global-target policy ("remap" | "pairwise" | "auto");
    block_fusion=False keeps every gate as given inside passes; candidate=i
    plans only the planner's i-th candidate gate list (sharded plans cost
    several; each one's modelled time is reported under "candidates");
    overlap=True costs them for a transport that overlaps a pass with the
    exchange after it (the runtime does on NCCL / loopback); readout=True also
    generates (compiles, with fusion=2) every pass's readout variant."""
    arr, keep = pack_gates(gates)
    flags = (int(fusion) | (((GLOBAL_POLICY[policy] + 1) << 4) if policy else 0) | (0 if block_fusion else 0x100)
             | (0 if low_remap else 0x200) | (0x400 if key_check else 0)
             | (((remap_lookahead + 1) & 31) << 12 if remap_lookahead is not None else 0)
             | (((candidate + 1) & 7) << 17 if candidate is not None else 0) | (1 << 20 if overlap else 0)
             | (1 << 21 if readout else 0))
    cap = 1 << 26
    while True:
        buf = ctypes.create_string_buffer(cap)
        s = N.lib().qsim_plan_json(n, n_ranks, arr, len(gates), flags, buf, cap)
        if s == 0:
            return buf.value.decode()
        if s == 1 and cap < (1 << 30):
            cap *= 4
            continue
        raise QsimError(s, "qsim_plan_json")


def exchange_peers(n: int, n_ranks: int, rank: int, gpos: Sequence[int]):
    """Host-only routing of a K-pair remap: (peer rank per chunk value, own chunk value)."""
    K = len(gpos)
    g = (ctypes.c_int * max(1, K))(*gpos)
    peers = (ctypes.c_int * (1 << K))()
    selfv = ctypes.c_int()
    s = N.lib().qsim_exchange_peers(n, n_ranks, rank, g, K, peers, ctypes.byref(selfv))
    if s != 0:
        raise QsimError(s, "qsim_exchange_peers")
    return list(peers), selfv.value


class QSim:
    """One context of the engine.

    transport: "local" (1 shard on this GPU), "virtual" (n_ranks shards on
    this GPU, exchanged by device copies), "nccl" (one process per GPU),
    "loopback" (one rank of an SPMD group whose ranks are threads of this
    process on this GPU: the NCCL transport's code path, see run_loopback).
    """

    def __init__(self, n: int, n_ranks: int = 1, transport: str = "local", rank: int = 0,
                 device: Optional[int] = None, nccl_id: Optional[bytes] = None,
                 scratch_bytes: Optional[int] = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("QSim needs a CUDA device (no CPU fallback)")
        self.lib = N.lib()
        self.n, self.n_ranks = n, n_ranks
        tp = {"local": N.TRANSPORT_LOCAL, "virtual": N.TRANSPORT_VIRTUAL, "nccl": N.TRANSPORT_NCCL,
              "loopback": N.TRANSPORT_LOOPBACK}[transport]
        G = (n_ranks - 1).bit_length()
        self.M = n - G
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        cfg = N.qsim_config()
        cfg.n_qubits, cfg.n_ranks, cfg.rank, cfg.transport = n, n_ranks, rank, tp
        nsh = n_ranks if tp == N.TRANSPORT_VIRTUAL else 1
        # PyTorch owns the device memory: one complex128 shard (as float64 pairs) per shard
        self._shards = [torch.empty(2 << self.M, dtype=torch.float64, device=dev) for _ in range(nsh)]
        for i, t in enumerate(self._shards):
            cfg.shards[i] = t.data_ptr()
        if tp in (N.TRANSPORT_NCCL, N.TRANSPORT_LOOPBACK):
            sb = self.lib.qsim_scratch_bytes(n, n_ranks) if scratch_bytes is None else scratch_bytes
            self._scratch = torch.empty(max(16, sb), dtype=torch.uint8, device=dev)
            cfg.scratch, cfg.scratch_bytes = self._scratch.data_ptr(), sb
            if nccl_id is None:
                raise ValueError("nccl/loopback transport needs nccl_id (QSim.distributed, get_loopback_id)")
            for j in range(128):
                cfg.nccl_id[j] = nccl_id[j]
        self._stream = torch.cuda.Stream(device=dev)
        cfg.stream = self._stream.cuda_stream
        h = ctypes.c_void_p()
        self._check(self.lib.qsim_create_ext(ctypes.byref(cfg), ctypes.byref(h)), "qsim_create_ext", ctx=False)
        self.ctx = h

    @classmethod
    def distributed(cls, n: int, group=None, device: Optional[int] = None, **kw) -> "QSim":
        """SPMD creation under torch.distributed: rank 0 draws the NCCL unique
        id and broadcasts it over the process group."""
        import torch.distributed as dist
        ws, rk = dist.get_world_size(group), dist.get_rank(group)
        obj = [get_unique_id() if rk == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(n, n_ranks=ws, transport="nccl", rank=rk, device=device, nccl_id=obj[0], **kw)

    # ------------------------------------------------------------ plumbing
    def _check(self, s: int, what: str, ctx: bool = True):
        if s != 0:
            msg = self.lib.qsim_last_error(self.ctx).decode() if ctx else ""
            raise QsimError(s, f"{what}: {msg}")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.qsim_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self):
        return self._stream

    # ------------------------------------------------------------ gates
    def init_basis(self, index: int = 0):
        self._check(self.lib.qsim_init_basis(self.ctx, index), "qsim_init_basis")

    def apply_1q(self, q: int, u):
        self._check(self.lib.qsim_apply_1q(self.ctx, q, _u4(u)), "qsim_apply_1q")

    def apply_controlled(self, controls: Sequence[int], target: int, u):
        c = (ctypes.c_int * max(1, len(controls)))(*controls)
        self._check(self.lib.qsim_apply_controlled(self.ctx, c, len(controls), target, _u4(u)),
                    "qsim_apply_controlled")

    def apply_perm(self, controls: Sequence[int], targets: Sequence[int], perm):
        c = (ctypes.c_int * max(1, len(controls)))(*controls)
        t = (ctypes.c_int * max(1, len(targets)))(*targets)
        p = np.ascontiguousarray(perm, dtype=np.uint32)
        self._check(self.lib.qsim_apply_perm(self.ctx, c, len(controls), t, len(targets),
                                             p.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))),
                    "qsim_apply_perm")

    def apply_swap(self, a: int, b: int):
        self._check(self.lib.qsim_apply_swap(self.ctx, a, b), "qsim_apply_swap")

    def remap(self, local_qubits: Sequence[int], global_qubits: Sequence[int]):
        K = len(local_qubits)
        lq = (ctypes.c_int * max(1, K))(*local_qubits)
        gq = (ctypes.c_int * max(1, K))(*global_qubits)
        self._check(self.lib.qsim_remap(self.ctx, lq, gq, K), "qsim_remap")

    def run_circuit(self, gates: Sequence = None, packed=None):
        arr, keep = packed if packed is not None else pack_gates(gates)
        n = len(gates) if gates is not None else len(arr)
        self._check(self.lib.qsim_run_circuit(self.ctx, arr, n), "qsim_run_circuit")

    # ------------------------------------------------------------ readout
    def probabilities(self, qubits: Sequence[int]) -> np.ndarray:
        k = len(qubits)
        out = np.zeros(1 << k, dtype=np.float64)
        q = (ctypes.c_int * max(1, k))(*qubits)
        self._check(self.lib.qsim_probabilities(self.ctx, q, k, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
                    "qsim_probabilities")
        return out

    def norm(self) -> float:
        return float(self.probabilities([])[0])

    def expectations(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.float64)
        self._check(self.lib.qsim_expectations(self.ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
                    "qsim_expectations")
        return out

    def expectations_async(self, out) -> None:
        """Enqueue <Q_i> into `out` (a pinned CPU torch tensor of n float64,
        valid after sync()); the host can go on enqueuing work meanwhile."""
        if out.dtype != torch_float64() or out.numel() != self.n or out.device.type != "cpu" or not out.is_contiguous():
            raise ValueError("out must be a contiguous CPU float64 tensor of n elements")
        self._check(self.lib.qsim_expectations_async(self.ctx, ctypes.c_void_p(out.data_ptr())),
                    "qsim_expectations_async")

    def measure(self, qubits: Sequence[int], seed: int, shots: int) -> np.ndarray:
        k = len(qubits)
        out = np.zeros(max(1, shots), dtype=np.uint64)
        q = (ctypes.c_int * max(1, k))(*qubits)
        self._check(self.lib.qsim_measure(self.ctx, q, k, seed, shots,
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))), "qsim_measure")
        return out[:shots]

    def get_amplitudes(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - first
        out = np.zeros(count, dtype=np.complex128)
        self._check(self.lib.qsim_get_amplitudes(self.ctx, first, count,
                                                 out.ctypes.data_as(ctypes.POINTER(N.c128))),
                    "qsim_get_amplitudes")
        return out

    def sync(self):
        self._check(self.lib.qsim_sync(self.ctx), "qsim_sync")

    def layout(self) -> List[int]:
        out = (ctypes.c_int * self.n)()
        self._check(self.lib.qsim_get_layout(self.ctx, out), "qsim_get_layout")
        return list(out)

    def set_option(self, key: str, value: int):
        self._check(self.lib.qsim_set_option(self.ctx, key.encode(), int(value)), "qsim_set_option")

    def stats(self) -> dict:
        s = N.qsim_stats()
        self._check(self.lib.qsim_get_stats(self.ctx, ctypes.byref(s)), "qsim_get_stats")
        return s.as_dict()

    def reset_stats(self):
        self._check(self.lib.qsim_reset_stats(self.ctx), "qsim_reset_stats")

    def shard_tensors(self) -> list:
        """The torch tensors backing the shards (physical order, float64 pairs)."""
        return list(self._shards)
