"""CPU: the C-ABI library and the checker libraries load and export every declared symbol.

No compute call is made here (no GPU in the build container)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header, prefix="mgpu_"):
    src = open(os.path.join(ROOT, header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z0-9_]+)\s*\(", src)))


def _exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_libmgpu_exports_every_declared_symbol():
    import paper_1606_01216_b200 as mg
    so = mg.mgpu.LIB_PATH
    assert os.path.exists(so), "libmgpu.so must be built (make lib)"
    declared = _declared("include/mgpu.h")
    missing = [s for s in declared if s not in _exported(so)]
    assert not missing, missing
    assert sorted(mg.mgpu.EXPORTED) == declared
    lib = ctypes.CDLL(so)
    for s in declared:
        getattr(lib, s)


def test_plugin_exports_every_declared_symbol():
    """include/mor_cuda.h: the drop-in SolveBackend's C entry points (libmor_cuda.so)."""
    from paper_1606_01216_b200 import plugin
    if not os.path.exists(plugin.LIB_PATH):
        pytest.skip("libmor_cuda.so needs the reference headers (make shim)")
    declared = _declared("include/mor_cuda.h", "mor_cuda_")
    missing = [s for s in declared if s not in _exported(plugin.LIB_PATH)]
    assert not missing, missing
    assert sorted(plugin.EXPORTED) == declared
    lib = plugin.lib()
    for s in declared:
        getattr(lib, s)


def test_library_is_sm100a_only():
    import paper_1606_01216_b200 as mg
    out = subprocess.run(["cuobjdump", "--list-elf", mg.mgpu.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_context_creation_fails_loudly_without_gpu():
    import paper_1606_01216_b200 as mg
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(mg.CudaError):
        mg.Context(0)


def test_host_models_match_oracle(oracle):
    """Product-side generators (csrc/models.cpp) == oracle generators, bitwise (host code, no GPU)."""
    import numpy as np

    import paper_1606_01216_b200 as mg
    for a, b in zip(mg.model_hermite(50), oracle.hermite_generate(50)):
        np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
        np.testing.assert_array_equal(a.col_idx, b.col_idx)
        np.testing.assert_array_equal(a.values, b.values)
    for a, b in zip(mg.model_chain(60, consistent=True), oracle.chain_generate(60, consistent=True)):
        np.testing.assert_array_equal(a.values, b.values)


def test_oracle_library_loads():
    from oracle import ORACLE_SO
    lib = ctypes.CDLL(ORACLE_SO)
    for s in ["orc_spai_build", "orc_spai_update", "orc_spai_ls", "orc_pcg_solve", "orc_block_solve",
              "orc_shifted_operator", "orc_thin_qr", "orc_chain_apply"]:
        getattr(lib, s)


def test_library_loads_before_torch():
    """libmgpu.so links neither NCCL nor cuBLAS: loading it first must not hand torch a foreign
    libnccl.so.2 (NCCL is resolved at the first mgpu_comm_* call, comm.cu)."""
    code = ("import sys; sys.path.insert(0, %r); import paper_1606_01216_b200 as mg; mg.lib(); "
            "import torch; print('ok')" % ROOT)
    out = subprocess.run([__import__("sys").executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
    needed = subprocess.run(["readelf", "-d", os.path.join(ROOT, "paper_1606_01216_b200", "lib", "libmgpu.so")],
                            capture_output=True, text=True).stdout
    assert "nccl" not in needed and "cublas" not in needed
