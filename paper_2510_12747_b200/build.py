"""In-tree build of libfvsr_b200.so (sm_100a only) with nvcc.

    python -m paper_2510_12747_b200.build            # build if sources are newer
    python -m paper_2510_12747_b200.build --force

The .so lands next to this file (git-ignored, but it travels to the GPU box with the
repo snapshot).  One translation unit: csrc/fvsr_api.cu includes the kernels.

The product library is always built with the product flags only: no environment variable
changes what it contains.  Experiment builds (instrumentation macros) go through
``build_variant`` into ``variants/`` and are loaded only when FVSR_LIB names them.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfvsr_b200.so")
SRC = os.path.join(HERE, "csrc", "fvsr_api.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
VARIANTS = os.path.join(REPO, "variants")

FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]


def _sources():
    return glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(REPO, "include", "fvsr_b200.h")]


def source_hash() -> str:
    h = hashlib.sha256()
    for s in sorted(_sources()):
        with open(s, "rb") as f:
            h.update(os.path.basename(s).encode() + b"\0" + f.read())
    return h.hexdigest()


def stale(path: str = LIB) -> bool:
    """True when the library is missing or was built from other sources (content hash in a
    sidecar file, so copies that do not keep mtimes are not rebuilt needlessly)."""
    if not os.path.exists(path):
        return True
    try:
        with open(path + ".srchash") as f:
            return f.read().strip() != source_hash()
    except OSError:
        return True


def _nvcc(out: str, macros: dict, verbose: bool) -> str:
    cmd = [NVCC, *FLAGS, "-o", out + ".tmp", SRC]
    flags = " ".join("-D%s=%s" % (k, v) for k, v in sorted(macros.items()))
    for k, v in sorted(macros.items()):
        cmd.insert(1, "-D%s=%s" % (k, v))
    # the macro set is recorded in the library (fvsr_build_flags) so a loader can refuse it
    cmd.insert(1, '-DFVSR_BUILD_FLAGS="%s"' % flags)
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building %s" % os.path.basename(out))
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(out + ".tmp", out)
    with open(out + ".srchash", "w") as f:
        f.write(source_hash())
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    """The product library (product flags only)."""
    if not force and not stale():
        return LIB
    return _nvcc(LIB, {}, verbose)


def build_variant(name: str, macros: dict, verbose: bool = False) -> str:
    """An experiment build (e.g. {"FVSR_ATTN_INSTRUMENT": 1}) into variants/, never over the
    product library.  Load it with FVSR_LIB=<path>."""
    os.makedirs(VARIANTS, exist_ok=True)
    out = os.path.join(VARIANTS, "libfvsr_b200_%s.so" % name)
    return _nvcc(out, dict(macros), verbose)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
