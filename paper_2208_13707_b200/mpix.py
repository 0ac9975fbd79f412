"""ctypes binding of include/mpix.h — the Python face of the drop-in boundary.

This mirrors the reference's `streamix::Proc` surface
(proj/include/streamix/world.hpp:35-92) the way a maintainer would bind the
C ABI: one `World` of N ranks (world.hpp:132-159), `run_ranks` to drive
collective calls from one thread per rank (proj/src/world.cpp:78-84),
`Info` hints (info.hpp:16-31), streams, stream communicators and the
enqueue family. Errors raise `MPIXError` whose `.name` is the reference's
`to_string(Err)` name (proj/src/result.cpp:5-32).

The library is the in-tree `libmpix.so`; there is no fallback path: if the
library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Callable, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPIX_LIB_PATH: an instrumented build (tools/sanitize.sh, libmpix_tsan.so)
LIB_PATH = os.environ.get("MPIX_LIB_PATH") or os.path.join(_HERE, "libmpix.so")

# --- constants (include/mpix.h) ---------------------------------------------
MPI_SUCCESS = 0
MPI_BYTE, MPI_INT, MPI_DOUBLE, MPI_FLOAT, MPIX_BFLOAT16 = 1, 2, 3, 4, 5
MPI_SUM, MPI_MAX, MPI_MIN = 1, 2, 3
MPI_ANY_SOURCE = -1
MPI_ANY_TAG = -1
MPIX_ANY_INDEX = -1
MPI_REQUEST_NULL = 0

ERR_NAMES = [
    "OK", "POOL_EXHAUSTED", "NO_EXPLICIT_POOL", "PENDING_OPS", "IN_USE", "BAD_HINT",
    "INVALID_STREAM", "INVALID_COMM", "INVALID_RANK", "INVALID_COUNT", "INVALID_TAG",
    "INVALID_REQUEST", "INVALID_INDEX", "MULTIPLEX_COMM", "NOT_MULTIPLEX", "WILDCARD_DST",
    "EMPTY_LIST", "NOT_ENQUEUE_COMM", "STREAM_MISMATCH", "QUEUE_BUSY", "CONFIG_INVALID",
    "NOT_FOUND", "BAD_ENCODING",
]
ERR = {n: i for i, n in enumerate(ERR_NAMES)}
ERR.update({"CUDA_ERROR": 100, "NOT_INITIALIZED": 101, "UNSUPPORTED": 102,
            "INVALID_ARG": 103, "INVALID_TYPE": 104, "INVALID_OP": 105, "NO_MEM": 106,
            "TIMEOUT": 107, "DEVICE_PROTOCOL": 108, "NOT_CORESIDENT": 109})

_TORCH_DT = {}


class MPIXError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = code
        self.name = error_string(code)
        super().__init__(f"{where}: {self.name} ({code})" if where else f"{self.name} ({code})")


class MPIStatus(C.Structure):
    _fields_ = [("MPI_SOURCE", C.c_int), ("MPI_TAG", C.c_int), ("MPI_ERROR", C.c_int),
                ("source_index", C.c_int), ("count_bytes", C.c_uint64), ("truncated", C.c_int)]

    def as_dict(self) -> dict:
        """The reference's Status (request.hpp:13-19) fields."""
        return {"source": self.MPI_SOURCE, "tag": self.MPI_TAG, "source_index": self.source_index,
                "bytes": self.count_bytes, "truncated": bool(self.truncated)}


_lib = None
_lib_lock = threading.Lock()
_owned_streams: list = []  # streams made by testing.new_stream (live for the process)

# Every spinning wait runs inside a stream-ordered kernel. CUDA multiplexes
# streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware queues (default 8); a
# stream blocked behind its own spinning Waitall would also hold back other
# streams sharing its queue, including the peers it waits for. Use the
# maximum (32) unless the user chose otherwise; it must be set before the
# CUDA context exists (DESIGN.md §6 "Hardware queues").
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def lib() -> C.CDLL:
    """Load libmpix.so (raises if it was not built: no CPU fallback exists)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib


def _declare(L: C.CDLL) -> None:
    P, I, U64, U32 = C.c_void_p, C.c_int, C.c_uint64, C.c_uint32
    sig = {
        "MPIX_Error_string": (C.c_char_p, [I]),
        "MPIX_World_init": (I, [I, P]),
        "MPIX_World_init_mp": (I, [I, I, P, P, P]),
        "MPIX_World_local_rank": (I, [C.POINTER(I)]),
        "MPIX_Heap_create": (I, [I, I, I, U64, U64, C.POINTER(U64), C.POINTER(U64), C.POINTER(I)]),
        "MPIX_Heap_attach": (I, [I, I]),
        "MPIX_Heap_contains": (I, [P, U64]),
        "MPIX_Heap_destroy": (I, []),
        "MPIX_Alloc_mem": (I, [U64, C.POINTER(P)]),
        "MPIX_Free_mem": (I, [P]),
        "MPIX_World_finalize": (I, []),
        "MPIX_World_size": (I, [C.POINTER(I)]),
        "MPIX_World_comm": (I, [I, C.POINTER(P)]),
        "MPIX_Rank_bind": (I, [I]),
        "MPIX_Comm_world_self": (I, [C.POINTER(P)]),
        "MPI_Comm_rank": (I, [P, C.POINTER(I)]),
        "MPI_Comm_size": (I, [P, C.POINTER(I)]),
        "MPI_Barrier": (I, [P]),
        "MPI_Comm_free": (I, [C.POINTER(P)]),
        "MPI_Info_create": (I, [C.POINTER(P)]),
        "MPI_Info_free": (I, [C.POINTER(P)]),
        "MPI_Info_set": (I, [P, C.c_char_p, C.c_char_p]),
        "MPI_Info_get": (I, [P, C.c_char_p, I, C.c_char_p, C.POINTER(I)]),
        "MPIX_Info_set_hex": (I, [P, C.c_char_p, P, I]),
        "MPIX_Info_get_hex": (I, [P, C.c_char_p, P, I, C.POINTER(I)]),
        "MPIX_Stream_create": (I, [P, C.POINTER(P)]),
        "MPIX_Stream_free": (I, [C.POINTER(P)]),
        "MPIX_Stream_get_cuda": (I, [P, C.POINTER(P)]),
        "MPIX_Stream_comm_create": (I, [P, P, C.POINTER(P)]),
        "MPIX_Stream_comm_create_multiplex": (I, [P, I, C.POINTER(P), C.POINTER(P)]),
        "MPIX_Stream_comm_create_multiple": (I, [P, I, C.POINTER(P), C.POINTER(P)]),
        "MPIX_Send_enqueue": (I, [P, I, I, I, I, P]),
        "MPIX_Recv_enqueue": (I, [P, I, I, I, I, P, P]),
        "MPIX_Isend_enqueue": (I, [P, I, I, I, I, P, C.POINTER(U64)]),
        "MPIX_Irecv_enqueue": (I, [P, I, I, I, I, P, C.POINTER(U64)]),
        "MPIX_Wait_enqueue": (I, [C.POINTER(U64), P]),
        "MPIX_Waitall_enqueue": (I, [I, C.POINTER(U64), P]),
        "MPIX_Request_free": (I, [C.POINTER(U64)]),
        "MPIX_Allreduce_enqueue": (I, [P, P, I, I, I, P]),
        "MPIX_Reduce_enqueue": (I, [P, P, I, I, I, I, P]),
        "MPIX_Reduce_scatter_block_enqueue": (I, [P, P, I, I, I, P]),
        "MPIX_Bcast_enqueue": (I, [P, I, I, I, P]),
        "MPIX_Allgather_enqueue": (I, [P, I, I, P, I, I, P]),
        "MPIX_Alltoall_enqueue": (I, [P, I, I, P, I, I, P]),
        "MPIX_Barrier_enqueue": (I, [P]),
        "MPI_Send": (I, [P, I, I, I, I, P]),
        "MPI_Recv": (I, [P, I, I, I, I, P, P]),
        "MPI_Isend": (I, [P, I, I, I, I, P, C.POINTER(U64)]),
        "MPI_Irecv": (I, [P, I, I, I, I, P, C.POINTER(U64)]),
        "MPI_Wait": (I, [C.POINTER(U64), P]),
        "MPI_Waitall": (I, [I, C.POINTER(U64), P]),
        "MPIX_Stream_send": (I, [P, I, I, I, I, P, I, I]),
        "MPIX_Stream_recv": (I, [P, I, I, I, I, P, I, I, P]),
        "MPIX_Stream_isend": (I, [P, I, I, I, I, P, I, I, C.POINTER(U64)]),
        "MPIX_Stream_irecv": (I, [P, I, I, I, I, P, I, I, C.POINTER(U64)]),
        "MPIX_Launch_count": (U64, []),
        "MPIX_Config_get": (I, [C.POINTER(U64), C.POINTER(I), C.POINTER(I), C.POINTER(U64)]),
        "MPIX_Comm_get_ctx": (I, [P, C.POINTER(U32)]),
        "MPIX_Comm_is_enqueue": (I, [P, C.POINTER(I)]),
        "MPIX_Type_size": (I, [I]),
        "MPIX_Version": (C.c_char_p, []),
        "MPIX_Rank_error": (I, [I, C.POINTER(U64)]),
        "MPIX_Comm_check": (I, [P]),
        "MPIX_Device_coresident": (I, [I, C.POINTER(I)]),
        "MPIX_Comm_region": (I, [P, C.POINTER(P), C.POINTER(U64)]),
        "MPIX_Trace_read": (I, [I, P, I, C.POINTER(I)]),
        "MPIXT_Copy_to_host": (I, [P, P, U64]),
        "MPIXT_Fill_pattern": (I, [P, U64, U32, U32, P]),
        "MPIXT_Checksum": (I, [P, U64, P, P]),
        "MPIXT_Saxpy": (I, [I, C.c_float, P, P, P]),
        "MPIXT_Fill_values": (I, [P, U64, I, I, U32, P]),
        "MPIXT_Delay": (I, [U64, P]),
        "MPIXT_Empty": (I, [P]),
        "MPIXT_Iter_fill": (I, [P, U64, P, C.c_float, C.c_float, P]),
        "MPIXT_Iter_check": (I, [P, U64, P, C.c_float, C.c_float, P, P]),
        "MPIXT_Iter_bump": (I, [P, P]),
        "MPIXT_Graph_begin": (I, [P]),
        "MPIXT_Graph_end": (I, [P, C.POINTER(P)]),
        "MPIXT_Graph_launch": (I, [P, P]),
        "MPIXT_Graph_destroy": (I, [P]),
        "MPIXT_Fill_f32": (I, [P, U64, C.c_float, P]),
        "MPIXT_Halo_pack": (I, [P, I, I, I, I, P, P]),
        "MPIXT_Halo_unpack": (I, [P, I, I, I, I, P, P]),
        "MPIXT_Stencil7": (I, [P, P, I, I, I, C.c_float, C.c_float, P]),
        "MPIXT_Launch_count": (U64, []),
        "MPIXT_Preload": (I, []),
        "MPIXT_Msgrate": (I, [I, I, I, I, P, P, P, P, P, P, P]),
        "MPIXT_Fig3": (I, [I, I, I, I, P, P, P, P, P]),
        "MPIXT_Exchange": (I, [P, P, P, P, P, P, U64, I, P, P, I, I, P]),
        "MPIXT_Set_exclusion": (I, [I, P]),
        "MPIXT_Pingpong": (I, [P, P, P, P, U64, I, P, P, I, I, P, P]),
        "MPIXT_Pingpong_side": (I, [P, P, U64, I, I, I, P, P]),
        "MPIXT_Selfchain": (I, [P, P, P, I, I, P, P, P]),
        "MPIXT_Stream_window": (I, [P, P, U64, I, I, I, I, P, P, P]),
        "MPIXT_Empty_loop": (I, [I, P, P, P]),
        "MPIXT_Loopback": (I, [P, P, P, U64, I, P, P, P]),
        "MPIXT_Allreduce_loop": (I, [I, P, P, P, P, P, I, I, I, I, P, P]),
        "MPIXT_Halo_steps": (I, [I, I, I, P, P, P, P, P, P, P, C.c_float, C.c_float, P, P]),
        "MPIXT_Stencil7_box": (I, [P, P, I, I, I, I, I, I, I, I, I, C.c_float, C.c_float, P]),
        "MPIXT_Stencil7_shell": (I, [P, P, I, I, I, C.c_float, C.c_float, P]),
        "MPIXT_Halo_pack6": (I, [P, I, I, I, P, P]),
        "MPIXT_Halo_unpack6": (I, [P, I, I, I, P, P]),
        "MPIXT_Stream_create": (I, [I, C.POINTER(P)]),
        "MPIXT_Stream_create_prio": (I, [I, I, C.POINTER(P)]),
        "MPIXT_Stream_destroy": (I, [P]),
        "MPIXT_Reduce_only": (I, [I, I, P, P, I, I, I, I, P]),
        "MPIXT_Copy_timing": (I, [I]),
        "MPIXT_Copy_timing_read": (I, [C.POINTER(C.c_double), C.POINTER(I), C.POINTER(U64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


# Symbols declared by include/mpix.h and include/mpix_testing.h (checked by
# tests/test_abi.py against the headers).
def exported_symbols() -> List[str]:
    import re
    out = []
    root = os.path.dirname(_HERE)
    for h in ("mpix.h", "mpix_testing.h"):
        txt = open(os.path.join(root, "include", h)).read()
        out += re.findall(r"^\s*(?:const\s+char\s*\*|int|uint64_t)\s+\**(MPIX?T?_\w+)\s*\(", txt, re.M)
    return out


def error_string(code: int) -> str:
    return lib().MPIX_Error_string(code).decode()


def check(rc: int, where: str = "") -> None:
    if rc != MPI_SUCCESS:
        raise MPIXError(rc, where)


def type_size(dt: int) -> int:
    return lib().MPIX_Type_size(dt)


def launch_count() -> int:
    return lib().MPIX_Launch_count() + lib().MPIXT_Launch_count()


def rank_error(rank: int) -> int:
    v = C.c_uint64()
    check(lib().MPIX_Rank_error(rank, C.byref(v)))
    return v.value


def device_coresident(device: int = 0) -> bool:
    """MPIX_Device_coresident: can two spinning kernels of different streams
    of `device` run concurrently (False under ncu's kernel serialisation)?"""
    v = C.c_int()
    check(lib().MPIX_Device_coresident(device, C.byref(v)), "MPIX_Device_coresident")
    return bool(v.value)


def trace_read(rank: int, max_records: int = 4096):
    """Per-op trace records of `rank` (MPIX_TRACE=1) as dicts."""
    import struct
    buf = C.create_string_buffer(128 * max_records)
    n = C.c_int()
    check(lib().MPIX_Trace_read(rank, buf, max_records, C.byref(n)))
    out = []
    for i in range(n.value):
        f = struct.unpack_from("<16Q", buf.raw, 128 * i)
        out.append({"seq": f[0], "is_recv": f[1] & 15, "mode": (f[1] >> 4) & 15,
                    "inline": (f[1] >> 8) & 15, "action": (f[1] >> 12) & 15, "bytes": f[2],
                    "key": f[3], "t": list(f[4:10]), "g0": f[10], "g1": f[11],
                    "gt": list(f[12:16])})
    return out


def config() -> dict:
    e, o = C.c_uint64(), C.c_uint64()
    r, m = C.c_int(), C.c_int()
    check(lib().MPIX_Config_get(C.byref(e), C.byref(r), C.byref(m), C.byref(o)))
    return {"eager_bytes": e.value, "ring_slots": r.value, "max_ctas": m.value,
            "oneshot_max_bytes": o.value}


def _ptr(buf) -> int:
    """Device address of a torch tensor, or an int address."""
    if buf is None:
        return 0
    if isinstance(buf, int):
        return buf
    return buf.data_ptr()


def _stream_handle(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


# --- Info ---------------------------------------------------------------------
class Info:
    """MPI_Info with MPIX_Info_set_hex (info.cpp:37-59)."""

    def __init__(self, **kv):
        h = C.c_void_p()
        check(lib().MPI_Info_create(C.byref(h)), "MPI_Info_create")
        self.h = h
        for k, v in kv.items():
            self.set(k, v)

    def set(self, key: str, value: str) -> None:
        check(lib().MPI_Info_set(self.h, key.encode(), value.encode()), "MPI_Info_set")

    def set_hex(self, key: str, value: bytes) -> None:
        b = C.create_string_buffer(bytes(value), max(1, len(value)))
        check(lib().MPIX_Info_set_hex(self.h, key.encode(), b, len(value)), "MPIX_Info_set_hex")

    def get(self, key: str) -> Optional[str]:
        buf = C.create_string_buffer(4096)
        flag = C.c_int()
        check(lib().MPI_Info_get(self.h, key.encode(), 4096, buf, C.byref(flag)))
        return buf.value.decode() if flag.value else None

    def get_hex(self, key: str) -> bytes:
        n = C.c_int()
        check(lib().MPIX_Info_get_hex(self.h, key.encode(), None, 0, C.byref(n)), "get_hex")
        buf = C.create_string_buffer(max(1, n.value))
        check(lib().MPIX_Info_get_hex(self.h, key.encode(), buf, n.value, C.byref(n)), "get_hex")
        return buf.raw[: n.value]

    def free(self) -> None:
        if self.h:
            check(lib().MPI_Info_free(C.byref(self.h)))
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def cuda_stream_info(stream) -> Info:
    """info{type="cudaStream_t", value=hex(stream)} — PAPER.md:839-840."""
    info = Info(type="cudaStream_t")
    info.set_hex("value", _stream_handle(stream).to_bytes(C.sizeof(C.c_void_p), "little"))
    return info


# --- Streams ---------------------------------------------------------------------
class Stream:
    """MPIX_Stream (proc_stream.cpp:7-60)."""

    def __init__(self, info: Optional[Info] = None, _keep=None):
        h = C.c_void_p()
        check(lib().MPIX_Stream_create(info.h if info else None, C.byref(h)), "MPIX_Stream_create")
        self.h = h
        self._keep = _keep  # the torch stream object, kept alive

    @classmethod
    def from_cuda(cls, torch_stream, **hints) -> "Stream":
        """hints: extra info keys, e.g. mpix_matching="dynamic" (a comm over
        this stream then accepts ANY_SOURCE / ANY_TAG receives)."""
        info = cuda_stream_info(torch_stream)
        for k, v in hints.items():
            info.set(k, v)
        return cls(info, _keep=torch_stream)

    def free(self) -> None:
        check(lib().MPIX_Stream_free(C.byref(self.h)), "MPIX_Stream_free")


NULL_STREAM = None


# --- Communicators -----------------------------------------------------------------
class Request:
    __slots__ = ("h",)

    def __init__(self, h: int):
        self.h = h


class Comm:
    """One rank's view of a communicator (CommH, comm.hpp:38-41)."""

    def __init__(self, h: C.c_void_p):
        self.h = h

    @property
    def rank(self) -> int:
        r = C.c_int()
        check(lib().MPI_Comm_rank(self.h, C.byref(r)))
        return r.value

    @property
    def size(self) -> int:
        r = C.c_int()
        check(lib().MPI_Comm_size(self.h, C.byref(r)))
        return r.value

    @property
    def ctx(self) -> int:
        r = C.c_uint32()
        check(lib().MPIX_Comm_get_ctx(self.h, C.byref(r)))
        return r.value

    @property
    def is_enqueue(self) -> bool:
        r = C.c_int()
        check(lib().MPIX_Comm_is_enqueue(self.h, C.byref(r)))
        return bool(r.value)

    def region_bytes(self) -> bytes:
        """Debug: a host copy of this member's peer-mapped region."""
        b, n = C.c_void_p(), C.c_uint64()
        check(lib().MPIX_Comm_region(self.h, C.byref(b), C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().MPIXT_Copy_to_host(buf, b, n.value))
        return buf.raw

    # collective ------------------------------------------------------------------
    def stream_comm_create(self, stream: Optional[Stream]) -> "Comm":
        out = C.c_void_p()
        check(lib().MPIX_Stream_comm_create(self.h, stream.h if stream else None, C.byref(out)),
              "MPIX_Stream_comm_create")
        return Comm(out)

    def stream_comm_create_multiplex(self, streams: Sequence[Optional[Stream]]) -> "Comm":
        arr = (C.c_void_p * max(1, len(streams)))(*[s.h.value if s else None for s in streams])
        out = C.c_void_p()
        check(lib().MPIX_Stream_comm_create_multiplex(self.h, len(streams), arr, C.byref(out)),
              "MPIX_Stream_comm_create_multiplex")
        return Comm(out)

    def barrier(self) -> None:
        check(lib().MPI_Barrier(self.h), "MPI_Barrier")

    def free(self) -> None:
        check(lib().MPI_Comm_free(C.byref(self.h)), "MPI_Comm_free")

    # enqueue ---------------------------------------------------------------------
    def send_enqueue(self, buf, count: int, dt: int, dest: int, tag: int) -> None:
        check(lib().MPIX_Send_enqueue(_ptr(buf), count, dt, dest, tag, self.h), "MPIX_Send_enqueue")

    def recv_enqueue(self, buf, count: int, dt: int, source: int, tag: int) -> None:
        check(lib().MPIX_Recv_enqueue(_ptr(buf), count, dt, source, tag, self.h, None),
              "MPIX_Recv_enqueue")

    def isend_enqueue(self, buf, count: int, dt: int, dest: int, tag: int) -> Request:
        r = C.c_uint64()
        check(lib().MPIX_Isend_enqueue(_ptr(buf), count, dt, dest, tag, self.h, C.byref(r)),
              "MPIX_Isend_enqueue")
        return Request(r.value)

    def irecv_enqueue(self, buf, count: int, dt: int, source: int, tag: int) -> Request:
        r = C.c_uint64()
        check(lib().MPIX_Irecv_enqueue(_ptr(buf), count, dt, source, tag, self.h, C.byref(r)),
              "MPIX_Irecv_enqueue")
        return Request(r.value)

    def allreduce_enqueue(self, sendbuf, recvbuf, count: int, dt: int, op: int = MPI_SUM) -> None:
        sb = 1 if sendbuf == "in_place" else _ptr(sendbuf)
        check(lib().MPIX_Allreduce_enqueue(sb, _ptr(recvbuf), count, dt, op, self.h),
              "MPIX_Allreduce_enqueue")

    def reduce_enqueue(self, sendbuf, recvbuf, count: int, dt: int, op: int = MPI_SUM,
                       root: int = 0) -> None:
        sb = 1 if sendbuf == "in_place" else _ptr(sendbuf)
        rb = _ptr(recvbuf) if recvbuf is not None else None
        check(lib().MPIX_Reduce_enqueue(sb, rb, count, dt, op, root, self.h), "MPIX_Reduce_enqueue")

    def reduce_scatter_block_enqueue(self, sendbuf, recvbuf, recvcount: int, dt: int,
                                     op: int = MPI_SUM) -> None:
        sb = 1 if sendbuf == "in_place" else _ptr(sendbuf)
        check(lib().MPIX_Reduce_scatter_block_enqueue(sb, _ptr(recvbuf), recvcount, dt, op, self.h),
              "MPIX_Reduce_scatter_block_enqueue")

    def bcast_enqueue(self, buf, count: int, dt: int, root: int = 0) -> None:
        check(lib().MPIX_Bcast_enqueue(_ptr(buf), count, dt, root, self.h), "MPIX_Bcast_enqueue")

    def allgather_enqueue(self, sendbuf, recvbuf, count: int, dt: int) -> None:
        """count elements per member; sendbuf may be "in_place"."""
        sb = 1 if sendbuf == "in_place" else _ptr(sendbuf)
        check(lib().MPIX_Allgather_enqueue(sb, count, dt, _ptr(recvbuf), count, dt, self.h),
              "MPIX_Allgather_enqueue")

    def alltoall_enqueue(self, sendbuf, recvbuf, count: int, dt: int) -> None:
        """count elements per (sender, receiver) block."""
        check(lib().MPIX_Alltoall_enqueue(_ptr(sendbuf), count, dt, _ptr(recvbuf), count, dt,
                                          self.h), "MPIX_Alltoall_enqueue")

    def barrier_enqueue(self) -> None:
        check(lib().MPIX_Barrier_enqueue(self.h), "MPIX_Barrier_enqueue")

    # conventional (host-thread) p2p on GPU buffers ----------------------------
    def send(self, buf, count: int, dt: int, dest: int, tag: int) -> None:
        check(lib().MPI_Send(_ptr(buf), count, dt, dest, tag, self.h), "MPI_Send")

    def recv(self, buf, count: int, dt: int, source: int, tag: int) -> dict:
        st = MPIStatus()
        check(lib().MPI_Recv(_ptr(buf), count, dt, source, tag, self.h, C.byref(st)), "MPI_Recv")
        return st.as_dict()

    def check(self) -> None:
        """MPIX_Comm_check: raises MPIXError(TIMEOUT) once a kernel of this
        member's rank hit its watchdog (sticky)."""
        check(lib().MPIX_Comm_check(self.h), "MPIX_Comm_check")

    def isend(self, buf, count: int, dt: int, dest: int, tag: int) -> Request:
        r = C.c_uint64()
        check(lib().MPI_Isend(_ptr(buf), count, dt, dest, tag, self.h, C.byref(r)), "MPI_Isend")
        return Request(r.value)

    def irecv(self, buf, count: int, dt: int, source: int, tag: int) -> Request:
        r = C.c_uint64()
        check(lib().MPI_Irecv(_ptr(buf), count, dt, source, tag, self.h, C.byref(r)), "MPI_Irecv")
        return Request(r.value)

    # multiplex stream p2p ----------------------------------
    def stream_send(self, buf, count: int, dt: int, dest: int, tag: int, src_idx: int,
                    dst_idx: int) -> None:
        check(lib().MPIX_Stream_send(_ptr(buf), count, dt, dest, tag, self.h, src_idx, dst_idx),
              "MPIX_Stream_send")

    def stream_recv(self, buf, count: int, dt: int, source: int, tag: int, src_idx: int,
                    dst_idx: int) -> dict:
        st = MPIStatus()
        check(lib().MPIX_Stream_recv(_ptr(buf), count, dt, source, tag, self.h, src_idx, dst_idx,
                                     C.byref(st)), "MPIX_Stream_recv")
        return st.as_dict()

    def stream_isend(self, buf, count: int, dt: int, dest: int, tag: int, src_idx: int,
                     dst_idx: int) -> Request:
        r = C.c_uint64()
        check(lib().MPIX_Stream_isend(_ptr(buf), count, dt, dest, tag, self.h, src_idx, dst_idx,
                                      C.byref(r)), "MPIX_Stream_isend")
        return Request(r.value)

    def stream_irecv(self, buf, count: int, dt: int, source: int, tag: int, src_idx: int,
                     dst_idx: int) -> Request:
        r = C.c_uint64()
        check(lib().MPIX_Stream_irecv(_ptr(buf), count, dt, source, tag, self.h, src_idx, dst_idx,
                                      C.byref(r)), "MPIX_Stream_irecv")
        return Request(r.value)


def wait_enqueue(req: Request) -> None:
    h = C.c_uint64(req.h if req else 0)
    check(lib().MPIX_Wait_enqueue(C.byref(h), None), "MPIX_Wait_enqueue")


def wait(req: Request) -> dict:
    """MPI_Wait (host): the request is consumed; returns its status."""
    h = C.c_uint64(req.h if req else 0)
    st = MPIStatus()
    check(lib().MPI_Wait(C.byref(h), C.byref(st)), "MPI_Wait")
    return st.as_dict()


def waitall(reqs: Sequence[Optional[Request]]) -> list:
    arr = (C.c_uint64 * max(1, len(reqs)))(*[(r.h if r else 0) for r in reqs])
    sts = (MPIStatus * max(1, len(reqs)))()
    check(lib().MPI_Waitall(len(reqs), arr, sts), "MPI_Waitall")
    return [sts[i].as_dict() for i in range(len(reqs))]


def waitall_enqueue(reqs: Sequence[Optional[Request]]) -> None:
    arr = (C.c_uint64 * max(1, len(reqs)))(*[(r.h if r else 0) for r in reqs])
    check(lib().MPIX_Waitall_enqueue(len(reqs), arr, None), "MPIX_Waitall_enqueue")


# --- World ------------------------------------------------------------------------
class World:
    """N ranks in this process, rank r on GPU devices[r] (world.hpp:132-159)."""

    def __init__(self, nranks: int, devices: Optional[Sequence[int]] = None):
        arr = (C.c_int * nranks)(*devices) if devices is not None else None
        check(lib().MPIX_World_init(nranks, arr), "MPIX_World_init")
        self.n = nranks
        self.devices = list(devices) if devices is not None else None

    def comm(self, rank: int) -> Comm:
        h = C.c_void_p()
        check(lib().MPIX_World_comm(rank, C.byref(h)), "MPIX_World_comm")
        return Comm(h)

    def run_ranks(self, fn: Callable[[int], object]) -> list:
        """fn(rank) once per rank on its own thread; re-raises the first error
        (proj/src/world.cpp:78-84)."""
        out = [None] * self.n
        errs = []

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        return out

    def finalize(self) -> None:
        check(lib().MPIX_World_finalize(), "MPIX_World_finalize")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.finalize()


# --- multi-process world (one process per GPU) ---------------------------------
_AG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p)

_TORCH_DTYPESTR = {}


class _RawCuda:
    """A raw device range exposed through __cuda_array_interface__."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class MPWorld:
    """This process hosts one rank of a world of torch.distributed's size
    (MPIX_World_init_mp): the symmetric heap is created and every peer's slice
    mapped (file descriptors passed over Unix sockets), and the runtime's
    collective host steps run over torch.distributed (gloo, CPU). Buffers
    that peers touch must come from `alloc`."""

    def __init__(self, heap_bytes: int = 4 << 30, device: Optional[int] = None):
        import socket
        import tempfile

        import torch
        import torch.distributed as dist
        assert dist.is_initialized(), "call torch.distributed.init_process_group first"
        self.dist, self.torch = dist, torch
        self.rank, self.n = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
        self.device = device
        torch.cuda.set_device(device)
        L = lib()
        base, slc, fd = C.c_uint64(), C.c_uint64(), C.c_int()
        ok = False
        for k in range(32):  # a virtual range free in every process
            cand = 0x600000000000 + (k << 40)
            rc = L.MPIX_Heap_create(self.rank, self.n, device, heap_bytes, cand, C.byref(base),
                                    C.byref(slc), C.byref(fd))
            flag = torch.tensor([1 if rc == 0 else 0])
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag[0]):
                ok = True
                break
            if rc == 0:
                L.MPIX_Heap_destroy()
        if not ok:
            raise MPIXError(ERR["NO_MEM"], "MPIX_Heap_create: no common virtual range")
        self.base, self.slice = base.value, slc.value
        # pass every rank's heap file descriptor to every other rank
        token = torch.randint(0, 2**31 - 1, (1,))
        dist.broadcast(token, 0)
        tmp = tempfile.gettempdir()
        path = lambda q: os.path.join(tmp, f"mpix_heap_{int(token[0])}_{q}")
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path(self.rank))
        srv.listen(self.n)
        dist.barrier()
        for q in range(self.n):
            if q != self.rank:
                c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                c.connect(path(q))
                socket.send_fds(c, [self.rank.to_bytes(4, "little")], [fd.value])
                c.close()
        for _ in range(self.n - 1):
            conn, _ = srv.accept()
            msg, fds, _, _ = socket.recv_fds(conn, 4, 1)
            check(L.MPIX_Heap_attach(int.from_bytes(msg, "little"), fds[0]), "MPIX_Heap_attach")
            os.close(fds[0])
            conn.close()
        srv.close()
        os.unlink(path(self.rank))
        os.close(fd.value)
        dist.barrier()
        devs = torch.zeros(self.n, dtype=torch.int64)
        mine = torch.tensor([device], dtype=torch.int64)
        parts = [torch.zeros(1, dtype=torch.int64) for _ in range(self.n)]
        dist.all_gather(parts, mine)
        devs = (C.c_int * self.n)(*[int(p[0]) for p in parts])

        def _allgather(inp, nbytes, out, ctx):
            try:
                b = torch.frombuffer(bytearray(C.string_at(inp, nbytes)), dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.n)]
                dist.all_gather(outs, b)
                joined = torch.cat(outs).numpy().tobytes()
                C.memmove(out, joined, len(joined))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._ag = _AG_FN(_allgather)  # keep the callback alive
        check(L.MPIX_World_init_mp(self.rank, self.n, devs, self._ag, None), "MPIX_World_init_mp")

    def comm(self) -> Comm:
        """This rank's world communicator."""
        h = C.c_void_p()
        check(lib().MPIX_World_comm(self.rank, C.byref(h)), "MPIX_World_comm")
        return Comm(h)

    def alloc(self, numel: int, dtype=None):
        """A torch tensor in this rank's slice of the symmetric heap."""
        torch = self.torch
        dtype = dtype or torch.uint8
        esz = torch.tensor([], dtype=dtype).element_size()
        p = C.c_void_p()
        check(lib().MPIX_Alloc_mem(max(1, numel * esz), C.byref(p)), "MPIX_Alloc_mem")
        typestr = {torch.uint8: "|u1", torch.int32: "<i4", torch.int64: "<i8",
                   torch.float32: "<f4", torch.float64: "<f8", torch.bfloat16: "<V2"}[dtype]
        if dtype is torch.bfloat16:  # no bfloat16 typestr: view int16 storage
            t = torch.as_tensor(_RawCuda(p.value, numel, "<i2"), device=f"cuda:{self.device}")
            return t.view(torch.bfloat16)
        return torch.as_tensor(_RawCuda(p.value, numel, typestr), device=f"cuda:{self.device}")

    def finalize(self) -> None:
        self.torch.cuda.synchronize(self.device)
        self.dist.barrier()
        check(lib().MPIX_World_finalize(), "MPIX_World_finalize")
        self.dist.barrier()  # no peer still maps my slice
        check(lib().MPIX_Heap_destroy(), "MPIX_Heap_destroy")


# --- test/bench helper kernels (include/mpix_testing.h) ---------------------------
class testing:
    @staticmethod
    def new_stream(device: int = 0, priority: int = 0):
        """A fresh CUDA stream as a torch ExternalStream (torch.cuda.Stream()
        draws from a 32-entry pool per device and aliases beyond that; ranks
        on aliased streams would be serialised). priority < 0: higher than
        the default (clamped to the device's range)."""
        import torch
        h = C.c_void_p()
        check(lib().MPIXT_Stream_create_prio(device, priority, C.byref(h)), "MPIXT_Stream_create")
        s = torch.cuda.ExternalStream(h.value, device=torch.device("cuda", device))
        _owned_streams.append(h.value)
        return s

    @staticmethod
    def fill_pattern(buf, nbytes: int, seed: int, it: int, stream) -> None:
        check(lib().MPIXT_Fill_pattern(_ptr(buf), nbytes, seed, it, _stream_handle(stream)))

    @staticmethod
    def fill_values(buf, count: int, dt: int, value_set: int, rank: int, stream) -> None:
        check(lib().MPIXT_Fill_values(_ptr(buf), count, dt, value_set, rank, _stream_handle(stream)),
              "MPIXT_Fill_values")

    @staticmethod
    def checksum(buf, nbytes: int, out_dev, stream) -> None:
        check(lib().MPIXT_Checksum(_ptr(buf), nbytes, _ptr(out_dev), _stream_handle(stream)))

    @staticmethod
    def saxpy(n: int, a: float, x, y, stream) -> None:
        check(lib().MPIXT_Saxpy(n, a, _ptr(x), _ptr(y), _stream_handle(stream)))

    @staticmethod
    def delay(ns: int, stream) -> None:
        check(lib().MPIXT_Delay(ns, _stream_handle(stream)))

    @staticmethod
    def empty(stream) -> None:
        check(lib().MPIXT_Empty(_stream_handle(stream)))

    # --- CUDA-Graph helpers: replay-dependent data and raw stream capture ---
    @staticmethod
    def iter_fill(x, n: int, it_dev, a: float, b: float, stream) -> None:
        """x[i] = (*it_dev + 1) * a + b * (i % 7), in-stream."""
        check(lib().MPIXT_Iter_fill(_ptr(x), n, _ptr(it_dev), a, b, _stream_handle(stream)))

    @staticmethod
    def iter_check(x, n: int, it_dev, a: float, b: float, bad_dev, stream) -> None:
        """Adds the number of i with x[i] != (*it_dev + 1) * a + b * (i % 7) to *bad_dev."""
        check(lib().MPIXT_Iter_check(_ptr(x), n, _ptr(it_dev), a, b, _ptr(bad_dev),
                                     _stream_handle(stream)))

    @staticmethod
    def iter_bump(it_dev, stream) -> None:
        check(lib().MPIXT_Iter_bump(_ptr(it_dev), _stream_handle(stream)))

    @staticmethod
    def graph_begin(stream) -> None:
        check(lib().MPIXT_Graph_begin(_stream_handle(stream)), "cudaStreamBeginCapture")

    @staticmethod
    def graph_end(stream) -> int:
        h = C.c_void_p()
        check(lib().MPIXT_Graph_end(_stream_handle(stream), C.byref(h)), "cudaStreamEndCapture")
        return h.value

    @staticmethod
    def graph_launch(exec_h: int, stream) -> None:
        check(lib().MPIXT_Graph_launch(exec_h, _stream_handle(stream)), "cudaGraphLaunch")

    @staticmethod
    def graph_destroy(exec_h: int) -> None:
        check(lib().MPIXT_Graph_destroy(exec_h), "cudaGraphExecDestroy")

    @staticmethod
    def fill_f32(x, n: int, v: float, stream) -> None:
        check(lib().MPIXT_Fill_f32(_ptr(x), n, v, _stream_handle(stream)))

    @staticmethod
    def halo_pack(u, nx, ny, nz, face, buf, stream) -> None:
        check(lib().MPIXT_Halo_pack(_ptr(u), nx, ny, nz, face, _ptr(buf), _stream_handle(stream)))

    @staticmethod
    def halo_unpack(u, nx, ny, nz, face, buf, stream) -> None:
        check(lib().MPIXT_Halo_unpack(_ptr(u), nx, ny, nz, face, _ptr(buf), _stream_handle(stream)))

    @staticmethod
    def stencil7(u, out, nx, ny, nz, w0, w1, stream) -> None:
        check(lib().MPIXT_Stencil7(_ptr(u), _ptr(out), nx, ny, nz, w0, w1, _stream_handle(stream)))

    @staticmethod
    def stencil7_box(u, out, nx, ny, nz, box, w0, w1, stream) -> None:
        """box = (x0, x1, y0, y1, z0, z1), 1-based inclusive."""
        check(lib().MPIXT_Stencil7_box(_ptr(u), _ptr(out), nx, ny, nz, *box, w0, w1,
                                       _stream_handle(stream)), "Stencil7_box")

    @staticmethod
    def stencil7_shell(u, out, nx, ny, nz, w0, w1, stream) -> None:
        check(lib().MPIXT_Stencil7_shell(_ptr(u), _ptr(out), nx, ny, nz, w0, w1,
                                         _stream_handle(stream)))

    @staticmethod
    def halo_pack6(u, nx, ny, nz, bufs, stream) -> None:
        arr = (C.c_void_p * 6)(*[_ptr(b) for b in bufs])
        check(lib().MPIXT_Halo_pack6(_ptr(u), nx, ny, nz, arr, _stream_handle(stream)))

    @staticmethod
    def halo_unpack6(u, nx, ny, nz, bufs, stream) -> None:
        arr = (C.c_void_p * 6)(*[_ptr(b) for b in bufs])
        check(lib().MPIXT_Halo_unpack6(_ptr(u), nx, ny, nz, arr, _stream_handle(stream)))

    # native drivers (csrc/mpix_drivers.cpp) -------------------------------
    @staticmethod
    def msgrate(comms, streams, sbufs, rbufs, devices, P: int, S: int, W: int, batches: int) -> dict:
        n = P * S
        CA = (C.c_void_p * n)(*[c.h for c in comms])
        SA = (C.c_void_p * n)(*[_stream_handle(s) for s in streams])
        SB = (C.c_void_p * n)(*[_ptr(b) for b in sbufs])
        RB = (C.c_void_p * n)(*[_ptr(b) for b in rbufs])
        DV = (C.c_int * P)(*devices)
        hs = (C.c_double * 2)()
        ds = C.c_double()
        check(lib().MPIXT_Msgrate(P, S, W, batches, CA, SA, SB, RB, DV, hs, C.byref(ds)), "Msgrate")
        msgs = P * S * W * batches
        return {"messages": msgs, "enqueue_s": hs[0], "host_s": hs[1], "device_s": ds.value,
                "msgs_per_s": msgs / max(ds.value, hs[1])}

    @staticmethod
    def fig3(comms, bufs, devices, T: int, W: int, batches: int, nbytes: int) -> dict:
        """The reference's lock-regime message-rate bench (Fig. 3) over
        conventional p2p, under the world's current host exclusion."""
        CA = (C.c_void_p * (2 * T))(*[c.h for c in comms])
        BA = (C.c_void_p * (2 * T))(*[_ptr(b) for b in bufs])
        DV = (C.c_int * 2)(*devices)
        el = C.c_double()
        n = C.c_long()
        check(lib().MPIXT_Fig3(T, W, batches, nbytes, CA, BA, DV, C.byref(el), C.byref(n)), "Fig3")
        return {"threads": T, "window": W, "messages": n.value, "elapsed_s": el.value,
                "msgs_per_s": n.value / max(el.value, 1e-9)}

    @staticmethod
    def exchange(c0, c1, s0, r0, s1, r1, nbytes: int, iters: int, st0, st1, dev0: int = 0,
                 dev1: int = 0) -> float:
        """Bidirectional Isend/Irecv/Waitall_enqueue exchange between ranks 0
        and 1 (native threads); returns device seconds for `iters` steps."""
        ds = C.c_double()
        check(lib().MPIXT_Exchange(c0.h, c1.h, _ptr(s0), _ptr(r0), _ptr(s1), _ptr(r1), nbytes, iters,
                                   _stream_handle(st0), _stream_handle(st1), dev0, dev1,
                                   C.byref(ds)), "Exchange")
        return ds.value

    @staticmethod
    def set_exclusion(regime: int) -> int:
        """0 global lock, 1 per communicator, 2 serial contexts (lock-free)."""
        prev = C.c_int()
        check(lib().MPIXT_Set_exclusion(regime, C.byref(prev)), "Set_exclusion")
        return prev.value

    @staticmethod
    def pingpong(c0, c1, b0, b1, nbytes: int, iters: int, s0, s1, dev0: int = 0, dev1: int = 0):
        ds, hs = C.c_double(), C.c_double()
        check(lib().MPIXT_Pingpong(c0.h, c1.h, _ptr(b0), _ptr(b1), nbytes, iters,
                                   _stream_handle(s0), _stream_handle(s1), dev0, dev1,
                                   C.byref(ds), C.byref(hs)), "Pingpong")
        return ds.value, hs.value

    @staticmethod
    def pingpong_side(c, buf, nbytes: int, iters: int, peer: int, initiator: bool, stream):
        ds = C.c_double()
        check(lib().MPIXT_Pingpong_side(c.h, _ptr(buf), nbytes, iters, peer, int(initiator),
                                        _stream_handle(stream), C.byref(ds)), "Pingpong_side")
        return ds.value

    @staticmethod
    def stream_window(c, buf, nbytes: int, window: int, reps: int, peer: int, sender: bool, stream):
        """One side of the cfg2 streaming-bandwidth loop; (device s, host s)."""
        d, h = C.c_double(), C.c_double()
        check(lib().MPIXT_Stream_window(c.h, _ptr(buf), nbytes, window, reps, peer, int(sender),
                                        _stream_handle(stream), C.byref(d), C.byref(h)),
              "MPIXT_Stream_window")
        return d.value, h.value

    @staticmethod
    def selfchain(c, prod, cons, n: int, iters: int, stream):
        ds, hs = C.c_double(), C.c_double()
        check(lib().MPIXT_Selfchain(c.h, _ptr(prod), _ptr(cons), n, iters, _stream_handle(stream),
                                    C.byref(ds), C.byref(hs)), "Selfchain")
        return ds.value, hs.value

    @staticmethod
    def reduce_only(P: int, me: int, sbufs, rbufs, count: int, dt: int, op: int, twoshot: bool, stream):
        SB = (C.c_void_p * P)(*[_ptr(b) for b in sbufs])
        RB = (C.c_void_p * P)(*[_ptr(b) for b in rbufs])
        check(lib().MPIXT_Reduce_only(P, me, SB, RB, count, dt, op, int(twoshot),
                                      _stream_handle(stream)), "Reduce_only")

    @staticmethod
    def copy_timing(enable: bool) -> None:
        check(lib().MPIXT_Copy_timing(int(enable)))

    @staticmethod
    def copy_timing_read():
        """(summed ms, count, bytes moved) of the timed copy grids that
        actually copied (the second arriver's grid of each message)."""
        ms, n, b = C.c_double(), C.c_int(), C.c_uint64()
        check(lib().MPIXT_Copy_timing_read(C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    HALO_SEQ, HALO_PIPE, HALO_COMPUTE, HALO_EXCHANGE = 0, 1, 2, 3

    @staticmethod
    def halo_steps(blocks, steps: int, devices, mode: int = 1):
        """Native cfg5 driver over 8 workloads.HaloStencil blocks (one per
        rank); returns (device seconds, host seconds) for `steps` steps.
        mode: HALO_SEQ / HALO_PIPE (interior overlapped with the exchange) /
        HALO_COMPUTE (stencil only) / HALO_EXCHANGE (exchange only)."""
        assert len(blocks) == 8
        VP = C.c_void_p
        comms = (VP * 8)(*[b.comm.h for b in blocks])
        streams = (VP * 8)(*[_stream_handle(b.stream) for b in blocks])
        devs = (C.c_int * 8)(*devices)
        u = (VP * 8)(*[_ptr(b.u) for b in blocks])
        v = (VP * 8)(*[_ptr(b.v) for b in blocks])
        sb = (VP * 48)(*[_ptr(b.sbuf[d]) for b in blocks for d in range(6)])
        rb = (VP * 48)(*[_ptr(b.rbuf[d]) for b in blocks for d in range(6)])
        ds, hs = C.c_double(), C.c_double()
        b0 = blocks[0]
        check(lib().MPIXT_Halo_steps(b0.n, steps, mode, comms, streams, devs, u, v, sb, rb,
                                     b0.W0, b0.W1, C.byref(ds), C.byref(hs)), "Halo_steps")
        if steps % 2 and mode != 3:
            for b in blocks:
                b.u, b.v = b.v, b.u
        return ds.value, hs.value

    @staticmethod
    def loopback(c, src, dst, nbytes: int, iters: int, stream):
        ds, hs = C.c_double(), C.c_double()
        check(lib().MPIXT_Loopback(c.h, _ptr(src), _ptr(dst), nbytes, iters, _stream_handle(stream),
                                   C.byref(ds), C.byref(hs)), "Loopback")
        return ds.value, hs.value

    @staticmethod
    def allreduce_loop(comms, streams, devices, sbufs, rbufs, count: int, dt: int, iters: int,
                       op: int = MPI_SUM):
        P = len(comms)
        VP = C.c_void_p
        ds, hs = C.c_double(), C.c_double()
        check(lib().MPIXT_Allreduce_loop(
            P, (VP * P)(*[c.h for c in comms]), (VP * P)(*[_stream_handle(s) for s in streams]),
            (C.c_int * P)(*devices), (VP * P)(*[_ptr(b) for b in sbufs]),
            (VP * P)(*[_ptr(b) for b in rbufs]), count, dt, op, iters, C.byref(ds), C.byref(hs)),
            "Allreduce_loop")
        return ds.value, hs.value

    @staticmethod
    def empty_loop(iters: int, stream):
        ds, hs = C.c_double(), C.c_double()
        check(lib().MPIXT_Empty_loop(iters, _stream_handle(stream), C.byref(ds), C.byref(hs)))
        return ds.value, hs.value
