"""Generate tests/golden/*.json from the REFERENCE itself.

Run in the build container (needs /root/reference to compile
oracle/_ref/libstreamix_ref.so):  python tests/golden/make_golden.py

Every value below is produced by the unmodified reference library through
oracle/ref_driver.cpp; the tests compare the C restatement (oracle/) and the
product (libmpix.so) against these files, so they run on boxes where the
reference is absent.
"""
import ctypes as C
import itertools
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=0, sort_keys=True)
    print("wrote", name)


def main():
    R = O.ref()
    assert R is not None, "reference library not built"

    # result.cpp:5-32
    dump("err_names.json", [R.ref_err_name(i).decode() for i in range(23)])

    # test_info.cpp:60-76 generation, encoded by the reference
    n = 1000
    raw = np.zeros(32 * n, dtype=np.uint8)
    lens = np.zeros(n, dtype=np.int32)
    enc = C.create_string_buffer(65 * n)
    R.ref_hex_random_vectors(42, n, raw.ctypes.data, lens.ctypes.data, enc)
    vecs = []
    for i in range(n):
        b = raw[32 * i: 32 * i + lens[i]].tobytes()
        e = enc.raw[65 * i: 65 * i + 65].split(b"\0")[0].decode()
        vecs.append([b.hex(), e])
    # malformed values (test_info.cpp:41-49) decoded by the reference
    bad = {}
    for s in ["xyz", "abc", "aB", "", "dead", "0g"]:
        out = C.create_string_buffer(16)
        ln = C.c_size_t()
        bad[s] = R.ref_hex_decode(s.encode(), out, C.byref(ln))
    dump("hex.json", {"random_mt19937_64_42": vecs, "decode_codes": bad,
                      "get_hex_missing": R.ref_info_get_hex_missing()})

    # wire header: the test_wire.cpp:8-29 envelope plus random ones
    hdrs = []
    rng = random.Random(7)
    cases = [(0x01020304, 7, -2, 3, 0x0A0B0C0D, 0x1122334455667788, 9)]
    for _ in range(200):
        cases.append((rng.getrandbits(32), rng.getrandbits(32), rng.randint(-2**31, 2**31 - 1),
                      rng.randint(-2**31, 2**31 - 1), rng.randint(-2**31, 2**31 - 1),
                      rng.getrandbits(64), rng.getrandbits(64)))
    for c in cases:
        out = np.zeros(36, dtype=np.uint8)
        R.ref_encode_header(*c, out.ctypes.data)
        hdrs.append([list(c), out.tobytes().hex()])
    dump("wire.json", hdrs)

    # enqueue edge semantics (Appendix A)
    codes = np.zeros(20, dtype=np.int32)
    R.ref_enqueue_errors(codes.ctypes.data, 20)
    dump("enqueue_errors.json", [R.ref_err_name(int(c)).decode() for c in codes])

    # matching: reference_outcome over sampled programs x all interleavings
    rng = random.Random(11)
    alphabet = lambda r: [(1, 1 - r, 0), (1, 1 - r, 1), (1, r, 0), (0, 1 - r, 0), (0, 1 - r, 1),
                          (0, r, 0), (0, -1, 0), (0, 1 - r, -1), (0, -1, -1)]
    match_cases = []
    for _ in range(400):
        progs = [[rng.choice(alphabet(r)) for _ in range(rng.randint(0, 3))] for r in range(2)]
        if not progs[0] and not progs[1]:
            continue
        base = [0] * len(progs[0]) + [1] * len(progs[1])
        orders = sorted(set(itertools.permutations(base)))
        for o in orders[:6]:
            pairs = O.ref_match_reference(progs, list(o))
            match_cases.append({"progs": progs, "order": list(o),
                                "pairs": [[int(x) for x in row] for row in pairs]})
    pp, ex, dv = C.c_uint64(), C.c_uint64(), C.c_uint64()
    R.ref_interleaving_oracle(6, C.byref(pp), C.byref(ex), C.byref(dv))
    dump("matching.json", {"cases": match_cases,
                           "interleaving_oracle_6": [pp.value, ex.value, dv.value]})

    # composed allreduce through the reference's enqueue calls
    ar = []
    rng = np.random.default_rng(5)
    for P in (2, 3, 4):
        for dt, code in (("i32", 1), ("f32", 2), ("f64", 3), ("bf16", 4)):
            for op in (1, 2, 3):
                cnt = 37
                if dt == "i32":
                    ins = rng.integers(-2**31, 2**31, size=(P, cnt), dtype=np.int64).astype(np.int32)
                elif dt == "f32":
                    ins = rng.uniform(-1, 1, size=(P, cnt)).astype(np.float32)
                elif dt == "f64":
                    ins = rng.uniform(-1, 1, size=(P, cnt))
                else:
                    f = rng.uniform(-1, 1, size=(P, cnt)).astype(np.float32)
                    ins = np.array([[O.orc().orc_f32_to_bf16_rne(float(v)) for v in row] for row in f],
                                   dtype=np.uint16)
                ins = np.ascontiguousarray(ins)
                out = np.zeros_like(ins)
                R.ref_allreduce(P, cnt, code, op, ins.ctypes.data, out.ctypes.data, 1)
                for r in range(1, P):
                    assert out[r].tobytes() == out[0].tobytes()
                ar.append({"P": P, "dt": dt, "op": op, "count": cnt,
                           "inputs": ins.tobytes().hex(), "output": out[0].tobytes().hex()})
    dump("allreduce.json", ar)

    # cfg1: 1 MiB fp32 x[i] = float(i % 1024) * 0.5f, 200 round trips
    x = (np.arange(262144) % 1024).astype(np.float32) * np.float32(0.5)
    f0, f1 = C.c_uint64(), C.c_uint64()
    R.ref_pingpong(x.ctypes.data, x.nbytes, 200, C.byref(f0), C.byref(f1))
    dump("cfg1.json", {"count": 262144, "iters": 200, "fnv1a64_rank0": f0.value,
                       "fnv1a64_rank1": f1.value})


if __name__ == "__main__":
    main()
