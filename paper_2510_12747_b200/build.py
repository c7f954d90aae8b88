"""In-tree build of libfvsr_b200.so (sm_100a only) with nvcc.

    python -m paper_2510_12747_b200.build            # build if sources are newer
    python -m paper_2510_12747_b200.build --force

The .so lands next to this file (git-ignored, but it travels to the GPU box with the
repo snapshot).  One translation unit: csrc/fvsr_api.cu includes the kernels.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfvsr_b200.so")
SRC = os.path.join(HERE, "csrc", "fvsr_api.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]


def _sources():
    return glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(REPO, "include", "fvsr_b200.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", LIB + ".tmp", SRC]
    if os.environ.get("FVSR_ATTN_INSTRUMENT"):  # experiments: per-tile timelines, debug short-cuts
        cmd.insert(1, "-DFVSR_ATTN_INSTRUMENT=1")
    if os.environ.get("FVSR_FIXED_REF"):  # experiments: 0 = always start from -inf references
        cmd.insert(1, "-DFVSR_FIXED_REF=" + str(int(os.environ["FVSR_FIXED_REF"])))
    if os.environ.get("FVSR_ATTN_EXP"):  # experiments: bottleneck ablations (not attention)
        cmd.insert(1, "-DFVSR_ATTN_EXP=" + str(int(os.environ["FVSR_ATTN_EXP"])))
    # experiments: V stages / P buffers at NQ=64, test_wait-first barriers, polynomial exp2,
    # QK pacing lead, per-CTA timeline stamps, softmax register budget
    for k in ("FVSR_NV64", "FVSR_NP64", "FVSR_MBAR_TEST_FIRST", "FVSR_POLY_EXP", "FVSR_QK_LEAD",
              "FVSR_CTA_TIMELINE", "FVSR_REG_SOFTMAX"):
        if os.environ.get(k):
            cmd.insert(1, "-D%s=%d" % (k, int(os.environ[k])))
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfvsr_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
