"""Build libstarscreen_b200.so in-tree with nvcc for sm_100a.

The screen kernel (ss_screen.cu) is compiled with -fmad=false so that no
fp64 multiply-add is contracted (bit parity with NumPy);
the host template code with -ffp-contract=off for the same reason.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libstarscreen_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-Xptxas", "-v"]

SOURCES = {
    "ss_api.cpp": [],
    "ss_template.cpp": [],
    "ss_build.cu": [],
    "ss_screen.cu": ["-fmad=false"],
    "ss_post.cu": [],
    "ss_featureset.cu": ["-fmad=false"],
    "ss_ladder.cpp": [],
    "ss_ladder_screen.cu": ["-fmad=false"],
    "ss_match.cu": ["-fmad=false"],
    "ss_session.cpp": [],
}


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_cc() -> list:
    # the image exports CC=/opt/gcc/bin/gcc (no libgomp/spec files); use the system g++
    for cand in ("/usr/bin/g++",):
        if os.path.exists(cand):
            return ["-ccbin", cand]
    return []


def build(verbose: bool = False) -> str:
    """Compile every source and link.  Experiment hooks (not used by the
    product build): SS_EXTRA_NVCC adds flags (e.g. -DRINGS_GROUP=64),
    SS_ONLY=a.cu,b.cu recompiles only those sources and reuses the others'
    objects from build/."""
    nvcc = _nvcc()
    extra_all = os.environ.get("SS_EXTRA_NVCC", "").split()
    only = set(filter(None, os.environ.get("SS_ONLY", "").split(",")))
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    for src, extra in SOURCES.items():
        obj = os.path.join(objdir, src + ".o")
        if only and src not in only and os.path.exists(obj):
            objs.append(obj)
            continue
        cmd = [nvcc, *_host_cc(), *ARCH, *COMMON, *extra, *extra_all, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = OUT + ".tmp"
    cmd = [nvcc, *_host_cc(), *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, OUT)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
