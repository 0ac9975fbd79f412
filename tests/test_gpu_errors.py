"""GPU: the error behaviour of the enqueue path against the reference's own
outcomes (tests/golden/enqueue_errors.json, produced by the compiled
reference through oracle/ref_driver.cpp:199-315).

Each case below is the reference probe's case k, issued through the C ABI
of this library (all 20; cases 1 and 4 go through the conventional
host-thread p2p, MPI_Isend / MPI_Irecv on the world comm).
"""
import json
import os

import pytest
import torch

from paper_2208_13707_b200 import mpix
from tests.gpu_util import gpu_world, sync_all

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "enqueue_errors.json")))


def code_of(fn):
    try:
        fn()
        return "OK"
    except mpix.MPIXError as e:
        return e.name


def test_enqueue_error_codes_match_reference(monkeypatch):
    monkeypatch.setenv("MPIX_MATCHING", "dynamic")  # case 8 receives with wildcards
    got = {}
    with gpu_world(2) as (w, ctx):
        buf = torch.zeros(4, dtype=torch.int32, device=0)
        sink = torch.zeros(64, dtype=torch.int32, device=0)
        c0, c1 = ctx[0].comm, ctx[1].comm
        # 0: enqueue precedence rank -> tag -> count (proc_enqueue.cpp:8-20)
        got[0] = code_of(lambda: c0.send_enqueue(buf, -1, mpix.MPI_INT, 1, -1))
        # 1: conventional p2p precedence rank -> count -> tag (proc_p2p.cpp:9-14)
        got[1] = code_of(lambda: w.comm(0).isend(buf, -1, mpix.MPI_INT, 1, -1))
        # 4: a conventional receive's request in an enqueue wait (no queue)
        conv = w.comm(0).irecv(sink[32:], 4, mpix.MPI_INT, 1, 77)
        got[4] = code_of(lambda: mpix.waitall_enqueue([conv]))
        w.comm(1).send(buf, 4, mpix.MPI_INT, 0, 77)
        mpix.wait(conv)
        # 2, 3: Waitall of nothing / of a null request (proc_enqueue.cpp:121-123)
        got[2] = code_of(lambda: mpix.waitall_enqueue([]))
        got[3] = code_of(lambda: mpix.waitall_enqueue([None]))
        # 5, 6, 7: multiplex comm, serial-context stream comm, world comm
        mux, serial = {}, {}

        def mk(r):
            mux[r] = w.comm(r).stream_comm_create_multiplex([ctx[r].mstream])
            serial[r] = w.comm(r).stream_comm_create(mpix.Stream())

        w.run_ranks(mk)
        got[5] = code_of(lambda: mux[0].send_enqueue(buf, 1, mpix.MPI_INT, 1, 0))
        got[6] = code_of(lambda: serial[0].send_enqueue(buf, 1, mpix.MPI_INT, 1, 0))
        got[7] = code_of(lambda: w.comm(0).send_enqueue(buf, 1, mpix.MPI_INT, 1, 0))
        # 8: a wildcard receive is accepted; rank 1 satisfies it
        got[8] = code_of(lambda: c0.irecv_enqueue(sink, 4, mpix.MPI_INT, mpix.MPI_ANY_SOURCE,
                                                  mpix.MPI_ANY_TAG))
        c1.send_enqueue(buf, 4, mpix.MPI_INT, 0, 5)
        # 9: destination outside the comm
        got[9] = code_of(lambda: c0.send_enqueue(buf, 1, mpix.MPI_INT, 2, 0))
        # 10: Waitall over requests of two different streams
        s2 = {}

        def mk2(r):
            s2[r] = w.comm(r).stream_comm_create(mpix.Stream.from_cuda(mpix.testing.new_stream(0)))

        w.run_ranks(mk2)
        ra = c0.irecv_enqueue(sink[8:], 4, mpix.MPI_INT, 1, 40)
        rb = s2[0].irecv_enqueue(sink[16:], 4, mpix.MPI_INT, 1, 41)
        got[10] = code_of(lambda: mpix.waitall_enqueue([ra, rb]))
        c1.send_enqueue(buf, 4, mpix.MPI_INT, 0, 40)
        s2[1].send_enqueue(buf, 4, mpix.MPI_INT, 0, 41)
        mpix.wait_enqueue(ra)
        mpix.wait_enqueue(rb)
        # 19 (A9): waiting twice on the same request is ok / ok
        rc = c0.isend_enqueue(buf, 1, mpix.MPI_INT, 1, 42)
        e1 = code_of(lambda: mpix.wait_enqueue(rc))
        e2 = code_of(lambda: mpix.wait_enqueue(rc))
        got[19] = "OK" if e1 == "OK" and e2 == "OK" else "FAILED"
        c1.recv_enqueue(sink[24:], 1, mpix.MPI_INT, 0, 42)
        # 11-15: stream hints (proc_stream.cpp:11-33)
        def hint(**kv):
            info = mpix.Info()
            for k, v in kv.items():
                if isinstance(v, bytes):
                    info.set_hex(k, v)
                else:
                    info.set(k, v)
            return code_of(lambda: mpix.Stream(info))
        got[11] = hint(type="bogus")
        got[12] = hint(type="cudaStream_t")
        got[13] = hint(type="cudaStream_t", value="zz")
        got[14] = hint(type="cudaStream_t", value=b"\x01\x02\x03")
        got[15] = hint(endpoint_policy="bogus")
        # 16: empty stream list
        got[16] = code_of(lambda: w.comm(0).stream_comm_create_multiplex([]))
        # 17, 18: freeing a stream in use / the null stream
        got[17] = code_of(lambda: ctx[0].mstream.free())
        got[18] = code_of(lambda: mpix.Stream.free(type("S", (), {"h": mpix.C.c_void_p()})()))
        sync_all(ctx)
        for r in range(2):
            torch.cuda.synchronize()
            assert mpix.rank_error(r) == 0
        assert int(sink[0]) == 0 and bool((sink[8:12] == 0).all())
    for k, name in got.items():
        assert name == GOLD[k], (k, name, GOLD[k])
    assert sorted(got) == list(range(20))


def test_wildcard_on_static_comm_is_unsupported(monkeypatch):
    """The one documented divergence: a static-matching comm rejects
    wildcards; the reference accepts them (case 8)."""
    monkeypatch.setenv("MPIX_MATCHING", "static")
    with gpu_world(1) as (w, ctx):
        t = torch.zeros(4, dtype=torch.int32, device=0)
        assert code_of(lambda: ctx[0].comm.irecv_enqueue(t, 4, mpix.MPI_INT, mpix.MPI_ANY_SOURCE,
                                                         0)) == "UNSUPPORTED"
