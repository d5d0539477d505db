"""The training step of the paper's large-vocabulary LM output path (§4.2, §6.4) through the
native step runtime of libtfs (include/tfs.h "Communicator" and "The training step";
csrc/step.cu).  Argument marshalling only: the stepper owns every buffer, orders every kernel
on its streams, runs the barriers and records the CUDA graph; this module creates it, exposes
its named buffers as torch tensors (views of the stepper's device memory), and -- in the
one-process-per-GPU mode -- all-gathers the communicator's IPC handles over torch.distributed
(plumbing).

    cfg  = StepConfig(vocab=800_000, dim=512, tokens=2560, num_sampled=8192)
    step = Step(cfg)                                  # R = 1
    E, W, b = step.tables(); E.copy_(...); ...; step.sync()
    loss = step.run(x, y)                             # device x, y int64 [B]
    step.capture(); loss = step.run(x, y)             # CUDA-graph replay

R > 1: ``Comm.distributed(cfg)`` (one process per GPU, torch.distributed initialised) or
``Comm.simulated(cfg)`` (all R ranks in this process on one GPU: the same phases, barriers
become stream ordering -- the single-GPU test mode), then ``Step(cfg, comm)``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import TFS_BF16, TFS_F32, TFS_REMOVE_ACCIDENTAL_HITS, TFS_SUBTRACT_LOG_Q, TfsError, check

OPTIMIZERS = {"sgd": 0, "momentum": 1, "adagrad": 2}

# named buffers (include/tfs.h TFS_BUF_*)
BUF = {name: i for i, name in enumerate((
    "E", "W", "b", "slot_E", "slot_W", "slot_b", "x", "y", "qw", "log_ec_s", "log_ec_y",
    "num_tries", "h", "w_rows", "b_rows", "loss", "lse", "loss_sum", "dh", "dw", "db", "err",
    "step", "counts"))}
_ROWS2D = {"E", "W", "slot_E", "slot_W", "h", "w_rows", "dh", "dw"}


@dataclass
class StepConfig:
    vocab: int
    dim: int
    tokens: int                 # B per replica
    num_sampled: int            # S per replica; 0 = full softmax (R > 1: vocabulary-sharded)
    num_shards: int = 1         # R
    lr: float = 0.1
    seed: int = 7
    unique: bool = True
    flags: int = TFS_SUBTRACT_LOG_Q | TFS_REMOVE_ACCIDENTAL_HITS
    operand_dtype: int = TFS_BF16
    optimizer: str = "sgd"      # "sgd" | "momentum" | "adagrad" (R-29)
    momentum: float = 0.9
    adagrad_init: float = 0.1
    cap_e: int = 0              # route slots per owner; 0 = worst case (never overflows)
    cap_w: int = 0

    @property
    def full_softmax(self) -> bool:
        return self.num_sampled == 0

    def c_struct(self):
        if self.optimizer not in OPTIMIZERS:
            raise ValueError(f"unknown optimizer {self.optimizer!r}")
        return _lib.StepConfigC(
            int(self.vocab), int(self.dim), int(self.num_shards), int(self.tokens),
            int(self.num_sampled), int(self.operand_dtype), int(self.flags), float(self.lr),
            int(bool(self.unique)), int(self.seed), OPTIMIZERS[self.optimizer],
            float(self.momentum), float(self.adagrad_init), int(self.cap_e), int(self.cap_w))


def heap_bytes(cfg: StepConfig) -> int:
    """Symmetric heap bytes per rank a step with this config needs (host arithmetic)."""
    return int(_lib.lib().tfs_step_heap_bytes(ctypes.byref(cfg.c_struct())))


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def device_tensor(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    """A torch view of `numel(shape)` elements of device memory at `ptr` (no copy)."""
    typestr = {torch.float32: "<f4", torch.int64: "<i8", torch.int32: "<i4",
               torch.bfloat16: "<i2", torch.uint8: "|u1"}[dtype]
    t = torch.as_tensor(_DevArray(ptr, shape, typestr), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def exchange_handles(handle: bytes, group=None) -> bytes:
    """All-gather every rank's 64-byte IPC handle in rank order (torch.distributed plumbing;
    gloo on CPU, NCCL on GPUs).  Returns R x 64 bytes."""
    import torch.distributed as dist
    assert len(handle) == 64
    R = dist.get_world_size(group)
    out = [None] * R
    dist.all_gather_object(out, handle, group=group)
    assert all(isinstance(h, bytes) and len(h) == 64 for h in out)
    return b"".join(out)


class Comm:
    """tfs_comm: symmetric device heap + device barriers (one per rank, or R simulated ranks)."""

    def __init__(self, ptr, R: int, first: int, nlocal: int, device):
        self.ptr, self.R, self.first, self.nlocal = ptr, R, first, nlocal
        self.device = torch.device(device)

    @classmethod
    def simulated(cls, cfg: StepConfig, device=None, timeout_ms: int = 0) -> "Comm":
        """All R = cfg.num_shards ranks in this process on one GPU (test / development mode):
        the same step phases; a barrier is stream ordering across the local ranks."""
        dev = torch.device(device or "cuda")
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        R = cfg.num_shards
        p = ctypes.c_void_p()
        check(_lib.lib().tfs_comm_create(R, 0, R, idx, heap_bytes(cfg), timeout_ms,
                                         ctypes.byref(p)), "tfs_comm_create")
        return cls(p, R, 0, R, torch.device("cuda", idx))

    @classmethod
    def distributed(cls, cfg: StepConfig, group=None, timeout_ms: int = 0) -> "Comm":
        """One process per GPU (torch.distributed initialised): this rank's heap, the IPC
        handles all-gathered, the peers' heaps mapped (NVLink P2P)."""
        import torch.distributed as dist
        R, rank = dist.get_world_size(group), dist.get_rank(group)
        assert R == cfg.num_shards, (R, cfg.num_shards)
        idx = torch.cuda.current_device()
        L = _lib.lib()
        p = ctypes.c_void_p()
        check(L.tfs_comm_create(R, rank, 1, idx, heap_bytes(cfg), timeout_ms, ctypes.byref(p)),
              "tfs_comm_create")
        h = ctypes.create_string_buffer(64)
        check(L.tfs_comm_export(p, h), "tfs_comm_export")
        allh = exchange_handles(h.raw, group)
        check(L.tfs_comm_connect(p, allh), "tfs_comm_connect")
        return cls(p, R, rank, 1, torch.device("cuda", idx))

    def barrier(self, channel: int = 15):
        """Device barrier on the current stream (one-process-per-GPU mode)."""
        check(_lib.lib().tfs_comm_barrier(self.ptr, int(channel), _stream()), "tfs_comm_barrier")

    def peer_bases(self, local: int = 0) -> torch.Tensor:
        """int64 [R] device tensor of the heap bases as seen from local rank `local`."""
        p = _lib.lib().tfs_comm_peer_bases(self.ptr, local)
        return device_tensor(p, (self.R,), torch.int64, self.device)

    def heap(self, local: int = 0) -> int:
        return int(_lib.lib().tfs_comm_heap(self.ptr, local) or 0)

    def error(self, local: int = 0):
        p = _lib.lib().tfs_comm_error(self.ptr, local)
        v = device_tensor(p, (2,), torch.int64, self.device).tolist()
        return int(v[0]) & 0xFFFFFFFF, int(v[1])

    def close(self):
        if self.ptr is not None:
            _lib.lib().tfs_comm_destroy(self.ptr)
            self.ptr = None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Step:
    """tfs_stepper: one synchronous step of every local rank (R = 1, or the comm's ranks)."""

    def __init__(self, cfg: StepConfig, comm: Comm | None = None, device=None):
        self.cfg = cfg
        self.comm = comm
        self.R = cfg.num_shards
        if self.R > 1 and comm is None:
            raise ValueError("R > 1 needs a Comm (Comm.distributed or Comm.simulated)")
        self.nlocal = comm.nlocal if comm is not None else 1
        self.first = comm.first if comm is not None else 0
        self.device = comm.device if comm is not None else torch.device(device or "cuda")
        p = ctypes.c_void_p()
        check(_lib.lib().tfs_step_create(ctypes.byref(cfg.c_struct()),
                                         comm.ptr if comm is not None else None,
                                         ctypes.byref(p)), "tfs_step_create")
        self.ptr = p
        self.B, self.d = cfg.tokens, cfg.dim
        self.c = 1.0 / (self.R * self.B)
        self.graph = False

    # ---- buffers
    def tensor(self, name: str, local: int = 0) -> torch.Tensor:
        """Named buffer of local rank `local` as a torch view (no copy)."""
        ptr, n, t = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int32()
        check(_lib.lib().tfs_step_buffer(self.ptr, local, BUF[name], ctypes.byref(ptr),
                                         ctypes.byref(n), ctypes.byref(t)), "tfs_step_buffer")
        dtype = (torch.float32, torch.bfloat16, torch.int64, torch.int32)[t.value]
        n = n.value
        if n == 0 or not ptr.value:
            return torch.empty(0, dtype=dtype, device=self.device)
        if name in _ROWS2D:
            shape = (n // self.d, self.d)
        elif name == "counts":
            shape = (2, self.R)
        else:
            shape = (n,)
        return device_tensor(ptr.value, shape, dtype, self.device)

    def tables(self, local: int = 0):
        return self.tensor("E", local), self.tensor("W", local), self.tensor("b", local)

    def slots(self, local: int = 0):
        return self.tensor("slot_E", local), self.tensor("slot_W", local), self.tensor("slot_b", local)

    def load_tables(self, E, W, b, local: int = 0):
        """Copy (this rank's shard of) E, W, b into the stepper's tables."""
        for dst, src in zip(self.tables(local), (E, W, b)):
            dst.copy_(torch.as_tensor(src).reshape(dst.shape))

    def sync(self):
        """After writing tables / slots: refresh derived copies, zero the error slots."""
        check(_lib.lib().tfs_step_sync(self.ptr), "tfs_step_sync")

    def set_step(self, value: int):
        """Set the step counter of every local rank (re-draws the sample drawn ahead)."""
        check(_lib.lib().tfs_step_set_counter(self.ptr, int(value)), "tfs_step_set_counter")

    # ---- running
    def run(self, x=None, y=None, timing_events=None):
        """One step of every local rank on the current stream.  x, y: device int64 tensors of
        nlocal * B ids (rank-major) or None (use the x / y buffers as they are).  Returns the
        loss_sum tensor of local rank 0 (device)."""
        io = _lib.StepIO()
        if x is not None:
            assert x.is_cuda and x.dtype == torch.int64 and x.numel() == self.nlocal * self.B
            assert y.is_cuda and y.dtype == torch.int64 and y.numel() == self.nlocal * self.B
            x, y = x.contiguous(), y.contiguous()
            io.x, io.y = x.data_ptr(), y.data_ptr()
        io.host = 0
        arr = None
        if timing_events is not None:
            for e in timing_events:  # torch creates its CUDA event lazily, at the first record
                if e is not None and not e.cuda_event:
                    e.record()
            arr = (ctypes.c_void_p * 21)(*[ctypes.c_void_p(e.cuda_event if e is not None else 0)
                                          for e in timing_events])
            io.timing_events = ctypes.cast(arr, ctypes.c_void_p)
        check(_lib.lib().tfs_step_run(self.ptr, ctypes.byref(io), _stream()), "tfs_step_run")
        return self.tensor("loss_sum", 0)

    def run_host(self, x_host, y_host, loss_host=None):
        """One step with HOST inputs (pinned int64 tensors of nlocal * B ids): the H2D copies,
        the step and the D2H copy of each local rank's loss_sum into loss_host (pinned float32
        [nlocal]) all happen inside the C call, on the current stream."""
        assert not x_host.is_cuda and x_host.dtype == torch.int64
        assert x_host.is_contiguous() and y_host.is_contiguous()
        io = _lib.StepIO()
        io.x, io.y = x_host.data_ptr(), y_host.data_ptr()
        io.host = 1
        io.loss_host = None if loss_host is None else loss_host.data_ptr()
        check(_lib.lib().tfs_step_run(self.ptr, ctypes.byref(io), _stream()), "tfs_step_run")
        return loss_host

    def capture(self):
        """Record one step of every local rank into a CUDA graph; later run() calls replay it."""
        check(_lib.lib().tfs_step_capture(self.ptr), "tfs_step_capture")
        self.graph = True

    def uncapture(self):
        check(_lib.lib().tfs_step_uncapture(self.ptr), "tfs_step_uncapture")
        self.graph = False

    def graph_kernels(self) -> int:
        return int(_lib.lib().tfs_step_graph_kernels(self.ptr))

    # ---- errors
    def error(self, local: int = 0):
        v = self.tensor("err", local).tolist()
        return int(v[0]) & 0xFFFFFFFF, int(v[1])

    def check(self, what: str = "step"):
        """Raise TfsError if any local rank's error slot (or the comm's) holds an error
        (reads device memory: synchronises)."""
        torch.cuda.synchronize(self.device)
        for l in range(self.nlocal):
            code, idx = self.error(l)
            if code == 0 and self.comm is not None:
                code, idx = self.comm.error(l)
            if code != 0:
                raise TfsError(code, f"{what} (rank {self.first + l})", idx)

    def close(self):
        if self.ptr is not None:
            torch.cuda.synchronize(self.device)
            _lib.lib().tfs_step_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
