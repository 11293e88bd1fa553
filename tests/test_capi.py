"""CPU-side checks of the C ABI boundary: the library builds for sm_100a, loads,
and exports every symbol declared in include/ffb200.h (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "ffb200.h")).read()
    return sorted(set(re.findall(r"^\S.*?\b(ffb_[a-z_0-9]+)\(", hdr, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1803_01982_b200 import _capi

    lib = _capi.load()
    declared = _declared()
    assert declared, "no declarations parsed"
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert set(_capi.EXPORTS) == set(declared)


def test_version_string():
    from paper_1803_01982_b200 import _capi

    assert b"sm_100a" in _capi.load().ffb_version()


def test_workspace_query_validates():
    from paper_1803_01982_b200 import _capi

    lib = _capi.load()
    p = _capi.Params(50, 60, 32, 10, 10, 0.5, 2.0, 0)
    nb = C.c_size_t()
    assert lib.ffb_workspace_query(2000, 1000, C.byref(p), _capi.FFB_MODE_FLIPFLOP, C.byref(nb)) == 0
    assert nb.value > 2000 * 1000 * 0  # sized
    bad = _capi.Params(50, 40, 32, 10, 10, 0.5, 2.0, 0)     # l < k
    assert lib.ffb_workspace_query(2000, 1000, C.byref(bad), 2, C.byref(nb)) == _capi.FFB_ERR_DIMENSION


def test_struct_layout_matches_header():
    from paper_1803_01982_b200 import _capi

    # ffb_params: 5 int64 + 2 double + uint64
    assert C.sizeof(_capi.Params) == 8 * 8
    r = _capi.Result
    assert r.alpha.offset == 8 * 20  # 20 pointer/int64 slots precede the host scalars


def test_sass_uses_fp64_tensor_cores():
    import subprocess

    lib = os.path.join(ROOT, "paper_1803_01982_b200", "libffb200.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "DMMA" in out, "GEMM engine must issue DMMA (FP64 tensor core) instructions"
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np

    import paper_1803_01982_b200 as ffb

    with pytest.raises(ffb.EngineUnavailable):
        ffb.flip_flop_srqr(np.eye(8), 3)


def test_sass_stages_tiles_with_tma():
    # the sketch / WT products load their tiles with cp.async.bulk.tensor (TMA)
    import subprocess

    lib = os.path.join(ROOT, "paper_1803_01982_b200", "libffb200.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTMALDG" in out


def test_batch_item_layout_matches_header():
    from paper_1803_01982_b200 import _capi

    # stream, mode(+pad), A, m, n, lda, a_layout(+pad), prm, omega, workspace, bytes, out, status
    assert _capi.BatchItem.a_layout.offset == 48
    assert _capi.BatchItem.prm.offset == 56


def test_import_requests_work_queues_without_overriding_the_caller():
    # batches run up to 16 problem streams: the package asks for 32 CUDA work
    # queues at import but never replaces a caller's setting
    import subprocess
    import sys

    code = "import os; import paper_1803_01982_b200; print(os.environ['CUDA_DEVICE_MAX_CONNECTIONS'])"
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.strip() == "32", out.stderr[-300:]
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "4"
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.strip() == "4"


def test_sass_has_cluster_async_stores_for_the_ring_jacobi():
    # the column-ring Jacobi hands boundary columns over with st.async + mbarrier
    # (SASS: STAS / SYNCS), no fence inside a sweep
    import subprocess

    lib = os.path.join(ROOT, "paper_1803_01982_b200", "libffb200.so")
    obj = os.path.join(ROOT, "paper_1803_01982_b200", "build", "ffb_jacobi_ring.o")
    sass = subprocess.run(["cuobjdump", "-sass", obj if os.path.exists(obj) else lib], capture_output=True, text=True).stdout
    assert "jacobi_ring_kernel" in sass
    assert "STAS" in sass and "SYNCS" in sass
