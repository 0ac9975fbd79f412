"""CPU: the C-ABI library loads, exports every symbol its headers declare,
and its host-side logic (error names, info/hex, hint validation, argument
checks before any CUDA call) matches the reference. No compute calls."""
import ctypes as C
import json
import os
import re
import subprocess

import pytest

from paper_2208_13707_b200 import mpix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    txt = "\n".join(l for l in txt.splitlines() if not l.lstrip().startswith("#"))
    return re.findall(r"\b((?:MPIX?T?_|MPI_)[A-Za-z0-9_]+)\s*\(", txt)


def test_library_exports_every_declared_symbol():
    syms = subprocess.run(["nm", "-D", "--defined-only", mpix.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    exported = {line.split()[-1] for line in syms.splitlines() if " T " in line}
    want = set(declared("mpix.h")) | set(declared("mpix_testing.h"))
    assert len(want) >= 45
    missing = sorted(want - exported)
    assert not missing, missing
    # nothing else leaks out of the library (version script)
    assert all(s.startswith(("MPI_", "MPIX_", "MPIXT_")) for s in exported), exported


def test_error_names_match_reference():
    names = json.load(open(os.path.join(GOLD, "err_names.json")))
    for code, name in enumerate(names):
        assert mpix.error_string(code) == name


def test_info_hex_matches_reference_vectors():
    g = json.load(open(os.path.join(GOLD, "hex.json")))
    info = mpix.Info()
    for raw, enc in g["random_mt19937_64_42"][:300]:
        b = bytes.fromhex(raw)
        info.set_hex("v", b)
        assert info.get("v") == enc
        assert info.get_hex("v") == b
    for s, code in g["decode_codes"].items():
        info.set("k", s)
        if code:
            with pytest.raises(mpix.MPIXError) as e:
                info.get_hex("k")
            assert e.value.code == code
        else:
            assert info.get_hex("k") == bytes.fromhex(s)
    with pytest.raises(mpix.MPIXError) as e:
        info.get_hex("missing")
    assert e.value.name == "NOT_FOUND"


def test_info_set_overwrites():  # test_info.cpp:51-58
    info = mpix.Info()
    info.set("k", "one")
    info.set_hex("k", b"\x7f")
    assert info.get("k") == "7f"


def _bad_hint(**kv):
    info = mpix.Info()
    for k, v in kv.items():
        if isinstance(v, bytes):
            info.set_hex(k, v)
        else:
            info.set(k, v)
    with pytest.raises(mpix.MPIXError) as e:
        mpix.Stream(info)
    return e.value.name


def test_stream_hint_validation_matches_reference():
    """proj/tests/test_stream.cpp:75-107 with type="cudaStream_t"."""
    e = json.load(open(os.path.join(GOLD, "enqueue_errors.json")))
    assert _bad_hint(type="exec_queue") == e[11] == "BAD_HINT"      # unknown type here
    assert _bad_hint(type="cudaStream_t") == e[12] == "BAD_HINT"    # missing value
    assert _bad_hint(type="cudaStream_t", value="zz") == e[13] == "BAD_HINT"
    assert _bad_hint(type="cudaStream_t", value=b"\x01\x02\x03") == e[14] == "BAD_HINT"
    assert _bad_hint(endpoint_policy="bogus") == e[15] == "BAD_HINT"
    # no type: a serial-context stream; policies accepted
    for pol in ("shared", "exclusive"):
        s = mpix.Stream(mpix.Info(endpoint_policy=pol))
        s.free()


def test_stream_free_null_is_invalid_stream():
    h = C.c_void_p()
    assert mpix.lib().MPIX_Stream_free(C.byref(h)) == mpix.ERR["INVALID_STREAM"]


def test_calls_without_world_fail_cleanly():
    L = mpix.lib()
    h = C.c_void_p()
    assert L.MPIX_World_comm(0, C.byref(h)) == mpix.ERR["NOT_INITIALIZED"]
    assert L.MPIX_Send_enqueue(None, 1, mpix.MPI_BYTE, 0, 0, None) == mpix.ERR["NOT_INITIALIZED"]
    arr = (C.c_uint64 * 1)(0)
    assert L.MPIX_Waitall_enqueue(0, arr, None) == mpix.ERR["NOT_INITIALIZED"]


def test_type_sizes():
    assert [mpix.type_size(t) for t in (1, 2, 3, 4, 5, 99)] == [1, 4, 8, 4, 2, 0]


def test_config_from_env_defaults():
    c = mpix.config()
    assert c["eager_bytes"] % 16 == 0 and c["ring_slots"] >= 2


def test_kernels_are_sm100a_sass():
    """The library carries sm_100a SASS for the runtime kernels (no PTX JIT)."""
    out = subprocess.run(["cuobjdump", "--list-elf", mpix.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_integration_c_example_compiles_and_links(tmp_path):
    """INTEGRATION.md's C example (Listing 2 against include/mpix.h)
    compiles for sm_100a and links against libmpix.so: the documented
    drop-in stays valid."""
    import shutil
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"## C example.*?```c\n(.*?)```", doc, flags=re.S)
    assert m, "C example block missing"
    src = tmp_path / "app.cu"
    src.write_text("__global__ void saxpy(int n, float a, const float* x, float* y) {\n"
                   "  int i = blockIdx.x * blockDim.x + threadIdx.x;\n"
                   "  if (i < n) y[i] = a * x[i] + y[i];\n}\n" + m.group(1) +
                   "\nint main() { int devs[2] = {0, 1}; return MPIX_World_init(2, devs) ? 1 : 0; }\n")
    libdir = os.path.dirname(mpix.LIB_PATH)
    r = subprocess.run([nvcc, "-gencode=arch=compute_100a,code=sm_100a", "-I" + os.path.join(ROOT, "include"),
                        str(src), "-o", str(tmp_path / "app"), "-L" + libdir, "-l:libmpix.so"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
