"""C-ABI boundary (CPU): the in-tree sm_100a library loads, exports exactly
the symbols include/rooflens_b200.h declares, and validates arguments the
way the reference models do -- without launching anything."""
import os
import re
import subprocess

import pytest

import paper_2502_16851_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rooflens_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^RL_API\s+[\w\s\*]+?\b(rl_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_the_binding_table():
    assert _declared() == P.EXPORTED_SYMBOLS


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", P.library_path], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (rl_\w+)$", out, flags=re.M)))
    assert exported == _declared()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", P.library_path], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_launch_counter():
    assert b"sm_100a" in P.lib().rl_version()
    assert P.kernel_launches() >= 0


def test_validation_errors_before_any_launch():
    L = P.lib()
    # precision other than FP64 -> ValidationError (reference ErrorKind 2)
    rc = L.rl_scale(P.CUDA_CORE, P.FP32, 1, 1, 1.0, 4, None, None)
    assert rc == 1 + 2 and L.rl_last_error().startswith(b"ValidationError: ")
    # n == 0 -> InvalidCount, exactly like scale_model (kernels.cpp:75-77)
    assert L.rl_scale(P.CUDA_CORE, P.FP64, 1, 1, 1.0, 0, None, None) == 1 + 5
    # null pointers
    assert L.rl_scale(P.CUDA_CORE, P.FP64, None, 1, 1.0, 4, None, None) == 1 + 2
    # unknown unit
    assert L.rl_scale(7, P.FP64, 1, 1, 1.0, 4, None, None) == 1 + 2
    # CSR: nnz = 0 is a ValidationError of the model
    assert L.rl_spmv_csr(P.CUDA_CORE, P.FP64, 4, 4, 0, 1, 1, 1, 1, 1, None, None) == 1 + 2
    # stencil: unknown preset, grid too small, steps 0, aliasing
    import ctypes as C
    dims = (C.c_uint64 * 3)(10, 10, 10)
    assert L.rl_stencil(0, 0, b"5d9pt", dims, None, 1, 1, 2, None, None) == 1 + 2
    small = (C.c_uint64 * 3)(2, 10, 1)
    assert L.rl_stencil(0, 0, b"2d5pt", small, None, 1, 1, 2, None, None) == 1 + 5
    assert L.rl_stencil(0, 0, b"2d5pt", dims, None, 0, 1, 2, None, None) == 1 + 5
    assert L.rl_stencil(0, 0, b"2d5pt", dims, None, 1, 1, 1, None, None) == 1 + 2
    # tensor-core formulation exists for 2d5pt / 3d7pt / 3d27pt only: checked
    # before the launch (the error names the restriction)
    assert L.rl_tuning_set(b"no_such_knob", 1, None) == 1 + 2


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    """An executing entry point on a machine without a device fails with a
    CUDA status (>= 100); it never computes on the host."""
    import ctypes as C
    buf = (C.c_double * 8)()
    rc = P.lib().rl_scale(P.CUDA_CORE, P.FP64, C.addressof(buf), C.addressof(buf), 2.0, 8, None, None)
    assert rc >= 100, rc
    assert b"CudaError" in P.lib().rl_last_error()


def test_every_documented_tuning_key_is_settable():
    """INTEGRATION.md's two tuning tables (product keys, developer keys) list
    exactly the keys rl_tuning_set accepts; setting one returns the previous
    value (restored here)."""
    import re

    text = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "INTEGRATION.md")).read()
    keys = []
    for head in ("| product key | selects |", "| family | keys |"):
        table = text[text.index(head):]
        end = table.find("\n\n")
        table = table if end < 0 else table[:end]
        keys += [k for row in table.splitlines()[2:] for k in re.findall(r"`([a-z0-9_]+)`", row.split("|")[1 if head.startswith("| product") else 2])]
    assert len(keys) >= 50 and len(set(keys)) == len(keys)
    for k in keys:
        prev = P.tuning_set(k, 1)
        assert P.tuning_set(k, prev) == 1, k
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2502_16851_b200", "csrc", "capi.cpp")).read()
    accepted = set(re.findall(r'\{"([a-z0-9_]+)", &rlb::Tuning::', src))
    assert accepted == set(keys)


def test_developer_tuning_keys_need_the_opt_in():
    """Without RL_DEV_TUNING=1 only the product keys are settable; launch-shape
    sweep knobs are refused with ValidationError (fresh process: the opt-in is
    read once)."""
    import subprocess
    import sys

    code = ("import paper_2502_16851_b200 as P\n"
            "P.tuning_set('stencil_tc3d_hybrid', 1)\n"
            "P.tuning_set('dist_graph', 1)\n"
            "try:\n    P.tuning_set('spmv_threads', 512)\nexcept P.RooflensError as e:\n"
            "    print(e.kind, 'developer sweep key' in str(e))\n")
    env = {k: v for k, v in os.environ.items() if k != "RL_DEV_TUNING"}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         check=True).stdout.split()
    assert out == ["ValidationError", "True"]
