"""INTEGRATION.md's rooflens-side adapter (integration/b200_exec.cpp),
compiled against the REFERENCE's own headers (/root/reference/proj/include)
and linked with the reference sources and librooflens_b200.so, then driven
by tests/integration_main.cpp: C statuses come back as rooflens::Error with
the reference's kind and text, and (no GPU here) an executing call reports a
CUDA status instead of falling back to the CPU.  Skipped where the reference
tree is absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "include")),
                                reason="reference tree absent")


@pytest.fixture(scope="module")
def probes(tmp_path_factory):
    out = tmp_path_factory.mktemp("integ") / "b200_exec_probe"
    libdir = os.path.join(ROOT, "paper_2502_16851_b200")
    srcs = [os.path.join(REF, "src", f) for f in sorted(os.listdir(os.path.join(REF, "src"))) if f.endswith(".cpp")]
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "integration"), "-I", NLOHMANN,
           os.path.join(ROOT, "integration", "b200_exec.cpp"), os.path.join(ROOT, "tests", "integration_main.cpp"),
           *srcs, "-L", libdir, "-lrooflens_b200", f"-Wl,-rpath,{libdir}", "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    import torch

    env = dict(os.environ)
    if not torch.cuda.is_available():
        env["RL_PROBE_NO_DEVICE"] = "1"
    res = subprocess.run([str(out)], check=True, capture_output=True, text=True, env=env)
    lines = {}
    for ln in res.stdout.splitlines():
        name, outcome = ln.split(" ", 1)
        lines[name] = outcome
    return lines


def test_unsupported_precision_is_a_validation_error(probes):
    assert probes["scale_fp32"].startswith("kind:2:ValidationError: precision FP32")
    assert probes["scale_null"].startswith("kind:2:ValidationError:")


def test_model_errors_match_the_reference(probes):
    # the adapter rethrows exactly what the reference model throws for the same arguments
    assert probes["spmv_bad_stats"] == probes["ref_spmv_bad_stats"]
    assert probes["stencil_unknown"] == probes["ref_stencil_unknown"]
    assert probes["spmv_bad_stats"].startswith("kind:2:")


def test_no_device_is_a_cuda_status_not_a_fallback(probes):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    assert probes["scale_exec"].startswith("runtime:CudaError")


def test_report_api_through_the_adapter(probes):
    """report.hpp's build_analysis / render_* (declared by the reference, no
    definition there) link against the adapter; its bounds are the
    reference's own bounds.cpp objects, value and text."""
    assert probes["report_bounds"] == "same"
    assert probes["report_alpha"] == "same"
    assert probes["report_min_depth"] == "3"  # 3d27pt: 3 * 3.375 > 9.99
    assert probes["report_verdict"].startswith("tensor cores cannot exceed 1.")
    assert int(probes["report_notes"]) == 2
    assert probes["render_json"] == "has_verdict"
    assert abs(float(probes["report_gemv_workload"]) - 1.05) < 1e-3
    assert int(probes["render_text_lines"]) >= 14
    assert probes["report_zero_balance"] == "kind:9"  # ZeroBalance


def test_plan_and_temporal_validation_through_the_adapter(probes):
    """SpmvPlan / stencil_temporal wrappers: malformed inputs raise the
    reference's ErrorKinds before any device allocation (no GPU needed)."""
    assert probes["plan_bad_column"].startswith("kind:14:IndexOutOfRange")
    assert probes["plan_decreasing_rows"].startswith("kind:2:ValidationError")
    assert probes["temporal_depth_9"].startswith("kind:10:InvalidRange")
