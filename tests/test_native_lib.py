"""The C-ABI library builds, loads without a GPU and exports exactly the
entry points include/cq.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_2505_06022_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "cq.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(cq_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(N.EXPORTED)


def test_library_exports_every_header_symbol():
    lib = N.load()
    for name in header_functions():
        assert hasattr(lib, name), name


def test_library_reports_missing_gpu_loudly():
    """Without a GPU every device call fails with a CUDA status -- there is
    no silent CPU path."""
    lib = N.load()
    n = ctypes.c_int32(-1)
    status = lib.cq_device_count(ctypes.byref(n))
    if status == N.CQ_OK and n.value > 0:
        pytest.skip("a GPU is visible")
    assert status != N.CQ_OK or n.value == 0
    with pytest.raises(Exception):
        import paper_2505_06022_b200 as cq
        from paper_2505_06022_b200 import workloads as W
        cq.run(cq.generate_commands(W.saxpy_program(64).graph(), 1))


def test_sm100a_code_in_library():
    """The fatbin carries sm_100a SASS (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_wave_kernels_have_no_contracted_fma():
    """The DSL rounds every operator, so the float32 wave kernels must not
    contain a scalar FFMA (ptxas contracts a packed mul feeding a packed add
    into FFMA2 even with --fmad=false; the kernels are written so it cannot).
    The fused kernels' FFMA2 are the deliberate, exact FMA form."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    lib = os.path.join(ROOT, "paper_2505_06022_b200", "libcq.so")
    sass = subprocess.run([tool, "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    wave = [f for f in funcs if re.match(r"_ZN2cq\d+wave5_\w*kernelIf", f)]
    assert len(wave) >= 4
    for f in wave:
        name = f.split("\n", 1)[0].strip()
        assert not re.search(r"\bFFMA\b(?!2)", f), name
        if "fused" not in name:
            assert "FFMA2" not in f, name


def test_no_cpu_fallback_without_the_library(monkeypatch):
    """The executor never computes on the CPU: without libcq.so a run raises
    (NativeError, a ClusterqError) instead of falling back."""
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import workloads as W
    monkeypatch.setattr(N, "LIB_PATH", os.path.join(ROOT, "no-such-dir", "libcq.so"))
    monkeypatch.setattr(N, "_lib", None)
    from paper_2505_06022_b200.scheduler import generate_commands_py
    prog = W.saxpy_program(1024, kind="float32")
    plan = generate_commands_py(prog.graph(), 2)
    with pytest.raises(cq.NativeError, match="no CPU fallback"):
        cq.run(plan)


def test_no_cpu_fallback_without_a_gpu():
    """With the library but no GPU (this container), a run fails loudly."""
    if os.path.exists("/dev/nvidiactl"):
        pytest.skip("a GPU is present")
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import workloads as W
    prog = W.saxpy_program(1024, kind="float32")
    with pytest.raises(cq.ClusterqError):
        cq.run(cq.generate_commands(prog.graph(), 1))


def test_torch_imports_after_libcq():
    """libcq and PyTorch share one libnccl.so.2 (the runpath prefers the NCCL
    wheel torch uses), so importing torch after libcq is loaded works."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2505_06022_b200 import _native as N\n"
            "N.load()\n"
            "import torch\n"
            "print('ok')\n") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
