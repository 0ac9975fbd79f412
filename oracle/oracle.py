"""ctypes access to the CPU oracle. TEST INFRASTRUCTURE ONLY.

- `orc()`: the C restatement of the reference (oracle/streamix_oracle.c)
- `ref()`: the UNMODIFIED reference library compiled from its own sources
  plus oracle/ref_driver.cpp (oracle/_ref/libstreamix_ref.so), or None when
  it was never built (e.g. a box that got no prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libstreamix_ref.so")

_orc = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            build()
        L = C.CDLL(ORC_SO)
        P, U64, I, SZ = C.c_void_p, C.c_uint64, C.c_int, C.c_size_t
        L.orc_err_name.restype = C.c_char_p
        L.orc_err_name.argtypes = [I]
        L.orc_hex_encode.argtypes = [P, SZ, C.c_char_p]
        L.orc_hex_decode.argtypes = [C.c_char_p, SZ, P, C.POINTER(SZ)]
        L.orc_encode_header.argtypes = [P, P]
        L.orc_decode_header.argtypes = [P, P]
        L.orc_wire_ctx.restype = C.c_uint32
        L.orc_wire_ctx.argtypes = [C.c_uint32, I]
        L.orc_check_enqueue_args.argtypes = [I, I, I, I, I]
        L.orc_check_p2p_args.argtypes = [I, I, I, I, I]
        L.orc_deliver.argtypes = [U64, U64, C.POINTER(U64), C.POINTER(I)]
        L.orc_match_reference.argtypes = [I, P, P, P, I, P, I]
        L.orc_match_static.argtypes = [I, P, P, P, I]
        for n in ("f32", "f64", "i32", "bf16"):
            getattr(L, f"orc_allreduce_{n}").argtypes = [P, I, SZ, I, P]
        L.orc_f32_to_bf16_rne.restype = C.c_uint16
        L.orc_f32_to_bf16_rne.argtypes = [C.c_float]
        L.orc_hash32.restype = C.c_uint32
        L.orc_hash32.argtypes = [U64, C.c_uint32]
        L.orc_exact_f32.restype = C.c_float
        L.orc_exact_f32.argtypes = [U64, C.c_uint32]
        L.orc_exact_bf16.restype = C.c_uint16
        L.orc_exact_bf16.argtypes = [U64, C.c_uint32]
        L.orc_pattern_u32.restype = C.c_uint32
        L.orc_pattern_u32.argtypes = [C.c_uint32, C.c_uint32, U64]
        L.orc_fill_pattern.argtypes = [P, U64, C.c_uint32, C.c_uint32]
        L.orc_checksum64.restype = U64
        L.orc_checksum64.argtypes = [P, U64]
        L.orc_fnv1a64.restype = U64
        L.orc_fnv1a64.argtypes = [P, U64]
        L.orc_stencil7.argtypes = [P, P, I, I, I, C.c_float, C.c_float]
        L.orc_halo_pack.argtypes = [P, I, I, I, I, P]
        L.orc_halo_unpack.argtypes = [P, I, I, I, I, P]
        L.orc_value_f32.restype = C.c_float
        L.orc_value_f32.argtypes = [U64, C.c_uint32, I]
        L.orc_value_bf16.restype = C.c_uint16
        L.orc_value_bf16.argtypes = [U64, C.c_uint32, I]
        L.orc_gen_checksum.restype = U64
        L.orc_gen_checksum.argtypes = [C.c_uint32, U64, I, I]
        L.orc_allreduce_gen.restype = U64
        L.orc_allreduce_gen.argtypes = [I, U64, I, I, I, I, P, P]
        L.orc_loopback_message.restype = U64
        L.orc_loopback_message.argtypes = [P, U64, P, U64, P]
        _orc = L
    return _orc


def ref():
    """The compiled reference, or None when unavailable."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/src"):
                build()
            if not os.path.exists(REF_SO):
                return None
        L = C.CDLL(REF_SO)
        P, U64, I, SZ, D = C.c_void_p, C.c_uint64, C.c_int, C.c_size_t, C.c_double
        L.ref_err_name.restype = C.c_char_p
        L.ref_err_name.argtypes = [I]
        L.ref_hex_encode.argtypes = [P, SZ, C.c_char_p]
        L.ref_hex_decode.argtypes = [C.c_char_p, P, C.POINTER(SZ)]
        L.ref_info_get_hex_missing.restype = I
        L.ref_encode_header.argtypes = [C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.c_int32,
                                        U64, U64, P]
        L.ref_hex_random_vectors.argtypes = [U64, I, P, P, P]
        L.ref_reference_outcome.argtypes = [I, P, P, P, I, P, I]
        L.ref_interleaving_oracle.argtypes = [I, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]
        L.ref_enqueue_errors.argtypes = [P, I]
        L.ref_pingpong.restype = D
        L.ref_pingpong.argtypes = [P, U64, I, C.POINTER(U64), C.POINTER(U64)]
        L.ref_selfmsg.restype = D
        L.ref_selfmsg.argtypes = [P, P, U64, I, I]
        L.ref_allreduce.restype = D
        L.ref_allreduce.argtypes = [I, U64, I, I, P, P, I]
        L.ref_msgrate.restype = D
        L.ref_msgrate.argtypes = [I, I, I, I, C.POINTER(U64)]
        L.ref_fig3.restype = D
        L.ref_fig3.argtypes = [I, I, I, I, C.POINTER(D)]
        _ref = L
    return _ref


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# --- numpy-level helpers over the C oracle --------------------------------------
def hex_encode(b: bytes) -> str:
    out = C.create_string_buffer(2 * len(b) + 1)
    src = C.create_string_buffer(bytes(b), max(1, len(b)))
    orc().orc_hex_encode(src, len(b), out)
    return out.value.decode()


def hex_decode(s: str):
    out = C.create_string_buffer(max(1, len(s) // 2))
    n = C.c_size_t()
    rc = orc().orc_hex_decode(s.encode(), len(s), out, C.byref(n))
    return rc, out.raw[: n.value] if rc == 0 else b""


def encode_header(ctx, src_rank, src_idx, dst_idx, tag, seq, length) -> bytes:
    env = np.zeros(1, dtype=np.dtype([("context_id", "<u4"), ("src_rank", "<u4"), ("src_idx", "<i4"),
                                      ("dst_idx", "<i4"), ("tag", "<i4"), ("pad", "<u4"),
                                      ("seq", "<u8"), ("payload_len", "<u8")]))
    env[0] = (ctx, src_rank, src_idx, dst_idx, tag, 0, seq, length)
    out = np.zeros(36, dtype=np.uint8)
    orc().orc_encode_header(_p(env), _p(out))
    return out.tobytes()


def _progs(programs):
    """programs: list per rank of (is_send, peer, tag) -> ctypes arrays."""
    n = len(programs)
    max_pos = max(1, max(len(p) for p in programs))
    arrays = [np.array(p if p else [(0, 0, 0)], dtype=np.int32).reshape(-1, 3) for p in programs]
    ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in arrays])
    lens = np.array([len(p) for p in programs], dtype=np.int32)
    return arrays, ptrs, lens, max_pos


def match_reference(programs, order):
    arrays, ptrs, lens, max_pos = _progs(programs)
    o = np.array(order, dtype=np.int32)
    pairs = np.zeros(len(programs) * max_pos, dtype=np.uint64)
    orc().orc_match_reference(len(programs), ptrs, _p(lens), _p(o), len(o), _p(pairs), max_pos)
    return pairs.reshape(len(programs), max_pos)


def match_static(programs):
    arrays, ptrs, lens, max_pos = _progs(programs)
    pairs = np.zeros(len(programs) * max_pos, dtype=np.uint64)
    orc().orc_match_static(len(programs), ptrs, _p(lens), _p(pairs), max_pos)
    return pairs.reshape(len(programs), max_pos)


def ref_match_reference(programs, order):
    arrays, ptrs, lens, max_pos = _progs(programs)
    flat = np.concatenate([np.array(p, dtype=np.int32).reshape(-1) for p in programs if p]) \
        if any(programs) else np.zeros(3, dtype=np.int32)
    o = np.array(order, dtype=np.int32)
    pairs = np.zeros(len(programs) * max_pos, dtype=np.uint64)
    ref().ref_reference_outcome(len(programs), _p(flat), _p(lens), _p(o), len(o), _p(pairs), max_pos)
    return pairs.reshape(len(programs), max_pos)


_AR = {"f32": (np.float32, "f32"), "f64": (np.float64, "f64"), "i32": (np.int32, "i32"),
       "bf16": (np.uint16, "bf16")}


def allreduce(inputs, dt: str, op: int = 1) -> np.ndarray:
    """Rank-ordered fold. inputs: list of P 1-D arrays (bf16 as uint16 bits)."""
    npdt, name = _AR[dt]
    ins = [np.ascontiguousarray(x, dtype=npdt) for x in inputs]
    n = ins[0].size
    out = np.zeros(n, dtype=npdt)
    ptrs = (C.c_void_p * len(ins))(*[x.ctypes.data for x in ins])
    getattr(orc(), f"orc_allreduce_{name}")(ptrs, len(ins), n, op, _p(out))
    return out


def fill_pattern(nbytes: int, seed: int, it: int) -> np.ndarray:
    out = np.zeros(max(1, nbytes), dtype=np.uint8)
    orc().orc_fill_pattern(_p(out), nbytes, seed, it)
    return out[:nbytes]


def checksum64(b: np.ndarray) -> int:
    b = np.ascontiguousarray(b).view(np.uint8)
    return int(orc().orc_checksum64(_p(b), b.size))


def fnv1a64(b: np.ndarray) -> int:
    b = np.ascontiguousarray(b).view(np.uint8)
    return int(orc().orc_fnv1a64(_p(b), b.size))


def exact_inputs(P: int, count: int, dt: str) -> list:
    """cfg3 exact value sets, vectorised (same hash as orc_hash32)."""
    i = np.arange(count, dtype=np.uint64)
    out = []
    for r in range(P):
        h = _hash32_np(i, r)
        if dt == "f32":
            out.append(((h % 2048).astype(np.int64) - 1024).astype(np.float32) / np.float32(256))
        else:
            f = ((h % 256).astype(np.int64) - 128).astype(np.float32) / np.float32(16)
            out.append((f.view(np.uint32) >> 16).astype(np.uint16))  # exact in bf16
    return out


_GEN_DT = {"f32": (1, np.float32), "bf16": (2, np.uint16)}


def value(i: int, r: int, dt: str, value_set: int):
    """One generated cfg3 input element (bf16 as uint16 bits)."""
    if dt == "f32":
        return np.float32(orc().orc_value_f32(i, r, value_set))
    return np.uint16(orc().orc_value_bf16(i, r, value_set))


def gen_checksum(r: int, count: int, dt: str, value_set: int) -> int:
    """checksum64 of rank r's generated input (count elements)."""
    return int(orc().orc_gen_checksum(r, count, _GEN_DT[dt][0], value_set))


def allreduce_gen(P: int, count: int, dt: str, value_set: int, op: int = 1, samples=()):
    """Rank-ordered allreduce of P generated inputs without materialising
    them: (checksum64 of the output, the output at `samples`)."""
    code, npdt = _GEN_DT[dt]
    idx = np.ascontiguousarray(np.asarray(samples, dtype=np.uint64))
    out = np.zeros(max(1, idx.size), dtype=npdt)
    cs = orc().orc_allreduce_gen(P, count, code, value_set, op, idx.size, _p(idx) if idx.size else None,
                                 _p(out))
    return int(cs), out[:idx.size]


def _hash32_np(i: np.ndarray, r: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = i * np.uint64(0x9E3779B97F4A7C15) + np.uint64((r * 0xD1B54A32D192ED03) % 2**64) + np.uint64(1)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def stencil7(u: np.ndarray, nx, ny, nz, w0, w1) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float32)
    out = u.copy()
    orc().orc_stencil7(_p(u), _p(out), nx, ny, nz, w0, w1)
    return out
