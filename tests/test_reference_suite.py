"""The reference's own unit tests for the hot path (P/tests/test_sparse.cpp, unmodified, 19
cases) built against the B200 operators: integration/vsr_b200_sparse.cpp replaces
P/src/sparse.cpp at link time (integration/Makefile, ref_test_sparse_b200), so
vsr::plan_sparse / sparse_attention_exec / sparsity_report run on the GPU.

  * CPU control (not gpu): the same test file linked with the reference's own sparse.o
    passes 19/19 -- the doctest shim (tests/doctest_shim) is faithful.
  * GPU: every partition, plan, accounting, row-range, determinism and error-taxonomy case
    passes unmodified (plans are bit-exact: fvsr_plan_sparse_f32 on the fp32 inputs).  The
    five cases that compare fp32 outputs at the reference's 1e-5 budget fail ONLY at those
    comparisons: the attention computes in bf16 on the tensor cores (tolerance stated in
    tests/helpers.py; measured per shape in profiles/parity_r2.json).
"""
import os
import re
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(os.path.dirname(HERE), "integration", "_build")
SRC = "test_sparse.cpp"

# case -> the reference source lines allowed to fail on the GPU (fp32 1e-5 output comparisons)
PRECISION_BOUND = {
    "saturated sparse exec equals the dense oracle": {212},
    "sparse exec equals a dense run restricted to selected pairs": {235},
    "diagonal-only plan with block-diagonal mask is per-block attention": {269},
    "sparse exec is independent of block visitation order": {291},
    "error versus dense decays as k grows": {360, 363},
}


def _run(binary):
    path = os.path.join(BUILD, binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built (make -C integration needs the reference tree)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    cases, cur = {}, None
    for line in r.stdout.splitlines():
        m = re.match(r"\[case\] (.*)", line)
        if m:
            cur = m.group(1)
            cases[cur] = {"status": None, "lines": set(), "other": []}
            continue
        m = re.match(r"\s+FAILED (\S+):(\d+): ", line)
        if m and cur:
            cases[cur]["lines"].add(int(m.group(2)))
            continue
        if line.strip().startswith("FAILED") and cur:
            cases[cur]["other"].append(line.strip())
            continue
        m = re.match(r"\[(PASS|FAIL)\] (.*)", line)
        if m:
            cases[m.group(2)]["status"] = m.group(1)
    return r, cases


def test_reference_suite_cpu_control():
    r, cases = _run("ref_test_sparse_cpu")
    assert len(cases) == 19 and all(c["status"] == "PASS" for c in cases.values()), r.stdout[-2000:]


@pytest.mark.gpu
def test_reference_suite_on_b200():
    r, cases = _run("ref_test_sparse_b200")
    assert len(cases) == 19, r.stdout[-3000:] + r.stderr[-2000:]
    for name, c in cases.items():
        if name in PRECISION_BOUND:
            assert not c["other"], (name, c["other"])
            assert c["lines"] <= PRECISION_BOUND[name], (name, sorted(c["lines"]))
        else:
            assert c["status"] == "PASS", (name, sorted(c["lines"]), c["other"], r.stdout[-3000:])
    passed = sum(c["status"] == "PASS" for c in cases.values())
    print(f"reference test_sparse.cpp on the B200: {passed}/19 cases pass unmodified")
