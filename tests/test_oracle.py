"""CPU: pin the oracle (oracle/streamix_oracle.c) to the reference.

Golden fixtures in tests/golden/ were produced by the unmodified reference
(tests/golden/make_golden.py); when the compiled reference is present
(oracle/_ref/) it is also cross-checked directly on fresh random inputs.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_err_names_match_reference():
    names = gold("err_names.json")
    assert [O.orc().orc_err_name(i).decode() for i in range(23)] == names


def test_hex_known_answers():
    # proj/tests/test_info.cpp:9-14, 16-23
    assert O.hex_encode(b"\xde\xad") == "dead"
    assert O.hex_encode(b"") == ""
    assert O.hex_decode("dead") == (0, b"\xde\xad")
    assert O.hex_decode("") == (0, b"")


def test_hex_vs_reference_vectors():
    g = gold("hex.json")
    assert len(g["random_mt19937_64_42"]) == 1000
    for raw, enc in g["random_mt19937_64_42"]:
        b = bytes.fromhex(raw)
        assert O.hex_encode(b) == enc
        assert len(enc) == 2 * len(b)  # test_info.cpp:72
        assert O.hex_decode(enc) == (0, b)
    for s, code in g["decode_codes"].items():
        assert O.hex_decode(s)[0] == code, s
    assert g["get_hex_missing"] == 21  # NOT_FOUND


def test_wire_header_golden_vector():
    # proj/tests/test_wire.cpp:21-29, verbatim expected bytes
    expect = bytes([0x04, 0x03, 0x02, 0x01, 0x07, 0x00, 0x00, 0x00, 0xfe, 0xff, 0xff, 0xff,
                    0x03, 0x00, 0x00, 0x00, 0x0d, 0x0c, 0x0b, 0x0a,
                    0x88, 0x77, 0x66, 0x55, 0x44, 0x33, 0x22, 0x11,
                    0x09, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00])
    assert O.encode_header(0x01020304, 7, -2, 3, 0x0A0B0C0D, 0x1122334455667788, 9) == expect


def test_wire_headers_vs_reference():
    for args, hexs in gold("wire.json"):
        assert O.encode_header(*args) == bytes.fromhex(hexs)


def test_wire_ctx():
    assert O.orc().orc_wire_ctx(5, 0) == 10 and O.orc().orc_wire_ctx(5, 1) == 11


def test_check_args_precedence():
    # Appendix A5: enqueue rank->tag->count vs p2p rank->count->tag
    e = gold("enqueue_errors.json")
    names = gold("err_names.json")
    assert names[O.orc().orc_check_enqueue_args(2, -1, 1, -1, 0)] == e[0] == "INVALID_TAG"
    assert names[O.orc().orc_check_p2p_args(2, -1, 1, -1, 0)] == e[1] == "INVALID_COUNT"
    assert names[O.orc().orc_check_enqueue_args(2, 1, 2, 0, 0)] == e[9] == "INVALID_RANK"
    assert O.orc().orc_check_enqueue_args(2, 4, -1, -1, 1) == 0  # A4 wildcards accepted


def test_deliver_truncation():
    import ctypes as C
    n, t = C.c_uint64(), C.c_int()
    O.orc().orc_deliver(100, 40, C.byref(n), C.byref(t))
    assert (n.value, t.value) == (40, 1)
    O.orc().orc_deliver(0, 40, C.byref(n), C.byref(t))
    assert (n.value, t.value) == (0, 0)


def test_matching_vs_reference_outcomes():
    g = gold("matching.json")
    assert len(g["cases"]) > 1000
    for c in g["cases"]:
        progs = [[tuple(op) for op in p] for p in c["progs"]]
        got = O.match_reference(progs, c["order"])
        exp = np.array(c["pairs"], dtype=np.uint64)
        assert np.array_equal(got[:, : exp.shape[1]], exp), c
    # the reference's exhaustive interleaving oracle (0 divergences)
    assert g["interleaving_oracle_6"] == [11108, 156016, 0]


def _all_programs(max_len, alphabet):
    out = [[]]
    for n in range(1, max_len + 1):
        out += [list(p) for p in itertools.product(alphabet, repeat=n)]
    return out


def test_static_seq_matching_equals_reference_for_concrete_patterns():
    """The product matches statically: k-th receive for (src, tag) <-> k-th
    send src->dst with that tag. For concrete patterns this
    must equal the reference matcher for EVERY interleaving."""
    cases = 0
    for r0 in _all_programs(3, [(1, 1, 0), (1, 1, 1), (1, 0, 0), (0, 1, 0), (0, 1, 1), (0, 0, 0)]):
        for r1 in _all_programs(2, [(1, 0, 0), (1, 0, 1), (0, 0, 0), (0, 0, 1), (1, 1, 0), (0, 1, 0)]):
            progs = [r0, r1]
            if not r0 and not r1:
                continue
            st = O.match_static(progs)
            base = [0] * len(r0) + [1] * len(r1)
            for o in set(itertools.permutations(base)):
                ref = O.match_reference(progs, list(o))
                assert np.array_equal(st, ref), (progs, o)
                cases += 1
    assert cases > 10000


def test_allreduce_vs_composed_reference():
    dts = {"i32": np.int32, "f32": np.float32, "f64": np.float64, "bf16": np.uint16}
    for c in gold("allreduce.json"):
        ins = np.frombuffer(bytes.fromhex(c["inputs"]), dtype=dts[c["dt"]]).reshape(c["P"], c["count"])
        got = O.allreduce(list(ins), c["dt"], c["op"])
        assert got.tobytes().hex() == c["output"], (c["P"], c["dt"], c["op"])


def test_exact_value_sets_are_order_independent():
    for dt in ("f32", "bf16"):
        ins = O.exact_inputs(8, 4096, dt)
        a = O.allreduce(ins, dt)
        b = O.allreduce(ins[::-1], dt)
        assert a.tobytes() == b.tobytes()
    # vectorised generator == the C generator
    assert O.exact_inputs(3, 5, "f32")[2][4] == np.float32(O.orc().orc_exact_f32(4, 2))
    assert O.exact_inputs(3, 5, "bf16")[1][3] == O.orc().orc_exact_bf16(3, 1)


def test_cfg1_checksum_golden():
    g = gold("cfg1.json")
    x = (np.arange(g["count"]) % 1024).astype(np.float32) * np.float32(0.5)
    assert O.fnv1a64(x) == g["fnv1a64_rank0"] == g["fnv1a64_rank1"]


def test_checksum_and_pattern_properties():
    b = O.fill_pattern(1003, 1, 2)
    assert b.size == 1003 and O.fill_pattern(1003, 1, 2).tobytes() == b.tobytes()
    assert O.fill_pattern(1003, 1, 3).tobytes() != b.tobytes()
    c = O.checksum64(b)
    b2 = b.copy()
    b2[500] ^= 1
    assert O.checksum64(b2) != c


def test_stencil_oracle_constant_field():
    nx = ny = nz = 6
    u = np.full((nz + 2) * (ny + 2) * (nx + 2), 2.0, dtype=np.float32)
    out = O.stencil7(u, nx, ny, nz, 0.5, 0.1)
    inner = out.reshape(nz + 2, ny + 2, nx + 2)[1:-1, 1:-1, 1:-1]
    assert np.allclose(inner, 0.5 * 2 + 0.1 * 12)


@pytest.mark.skipif(O.ref() is None, reason="compiled reference absent")
def test_live_cross_check_with_reference():
    import ctypes as C
    R = O.ref()
    rng = random.Random(3)
    for _ in range(200):
        b = bytes(rng.getrandbits(8) for _ in range(rng.randint(0, 40)))
        out = C.create_string_buffer(2 * len(b) + 1)
        R.ref_hex_encode(C.create_string_buffer(b, max(1, len(b))), len(b), out)
        assert out.value.decode() == O.hex_encode(b)
    rs = np.random.default_rng(9)
    for P in (2, 5):
        ins = np.ascontiguousarray(rs.uniform(-1, 1, (P, 301)).astype(np.float32))
        out = np.zeros_like(ins)
        R.ref_allreduce(P, 301, 2, 1, ins.ctypes.data, out.ctypes.data, 1)
        assert out[0].tobytes() == O.allreduce(list(ins), "f32").tobytes()


def test_generated_allreduce_oracle_equals_materialised_fold():
    """orc_allreduce_gen (cfg3 at full size, inputs generated per element)
    computes the same fold as orc_allreduce_f32/bf16 over materialised inputs,
    and its "exact" set is the exact_inputs value set."""
    for dt, npdt in (("f32", np.float32), ("bf16", np.uint16)):
        for vs in (0, 1):
            n, P = 4099, 3
            ins = [np.array([O.value(i, r, dt, vs) for i in range(n)], dtype=npdt) for r in range(P)]
            exp = O.allreduce(ins, dt)
            cs, samp = O.allreduce_gen(P, n, dt, vs, 1, [0, 7, n - 1])
            assert cs == O.checksum64(exp)
            assert samp.view(np.uint8).tobytes() == exp[[0, 7, n - 1]].view(np.uint8).tobytes()
            assert O.gen_checksum(2, n, dt, vs) == O.checksum64(ins[2])
            if vs == 0:
                for a, b in zip(O.exact_inputs(P, n, dt), ins):
                    assert a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes()
            else:  # uniform(-1, 1), order-sensitive: not every sum is exact
                f = ins[0].astype(np.float32) if dt == "f32" else (ins[0].astype(np.uint32) << 16).view(np.float32)
                assert f.min() >= -1.0 and f.max() <= 1.0  # bf16 RNE may reach 1.0


def test_model_check_enumeration_and_matching_follow_the_reference_matcher():
    """tests/model_check.py (the GPU bounded model check of SPEC.md:437):
    the enumeration size, and its expected pairs equal the reference
    matcher's (orc_match_reference, pinned to the reference in
    tests/golden/matching.json) on every program, per communicator, for the
    rank-0-first interleaving of each program's operations."""
    from tests import model_check as M
    progs = list(M.programs(2))
    done = [p for p, _ in progs if M.completes(p)]
    assert (len(progs), len(done)) == (9856, 6864)
    for prog in done[::7]:
        exp = M.expected_pairs(prog)
        for comm in (0, 1):
            rank_ops = [[], []]
            where = [[], []]
            for r in (0, 1):
                for pos, (kind, peer, tag, _) in enumerate(prog.get((r, comm), [])):
                    rank_ops[r].append((1 if kind in ("Send", "Isend") else 0, peer, tag))
                    where[r].append(pos)
            if not rank_ops[0] and not rank_ops[1]:
                continue
            order = [0] * len(rank_ops[0]) + [1] * len(rank_ops[1])
            pairs = O.match_reference(rank_ops, order)
            for r in (0, 1):
                for i, (is_send, _, _) in enumerate(rank_ops[r]):
                    if is_send:
                        continue
                    s = int(pairs[r][i])
                    sr, si = s >> 16, s & 0xFFFF
                    assert exp[(r, comm, where[r][i])] == (sr, comm, where[sr][si])


def test_reference_fig3_runs_every_regime():
    """The reference's own lock-regime bench (bench.cpp:118-235) through
    oracle/_ref: the CPU baseline bench.py reports beside MPIXT_Fig3."""
    import ctypes as C
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built")
    for mode in (0, 1, 2):
        m = C.c_double()
        assert R.ref_fig3(mode, 2, 16, 320, C.byref(m)) > 0
        assert m.value > 0
