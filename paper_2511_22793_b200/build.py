"""Build libgsparc_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2511_22793_b200.build        # incremental
    python -m paper_2511_22793_b200.build --force

Objects go to paper_2511_22793_b200/_build/, the shared library next to this
file (both git-ignored, both shipped to the GPU box by gpurun).
"""

from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libgsparc_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
         "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_digest():
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cuh", ".h")):
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()[:16]


def _compile(src, hdr, force):
    path = os.path.join(CSRC, src)
    with open(path, "rb") as fh:
        digest = hashlib.sha256(fh.read() + hdr.encode() +
                                " ".join(FLAGS + ARCH).encode()).hexdigest()[:16]
    obj = os.path.join(OBJ, f"{src[:-3]}.{digest}.o")
    if os.path.exists(obj) and not force:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    for stale in os.listdir(OBJ):
        if stale.startswith(src[:-3] + ".") and stale.endswith(".o") and \
                os.path.join(OBJ, stale) != obj:
            os.remove(os.path.join(OBJ, stale))
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force=False, verbose=True, experiments=False):
    """experiments=True compiles the timing/tuning environment knobs in
    (-DGSPARC_EXPERIMENTS, common.cuh experiment_env); the default product
    build ignores them."""
    global FLAGS
    FLAGS = [f for f in FLAGS if f != "-DGSPARC_EXPERIMENTS"]
    if experiments:
        FLAGS = FLAGS + ["-DGSPARC_EXPERIMENTS"]
    os.makedirs(OBJ, exist_ok=True)
    hdr = _headers_digest()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, force), _sources()))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--experiments", action="store_true",
                    help="compile in the GSPARC_* experiment knobs")
    a = ap.parse_args()
    build(force=a.force, experiments=a.experiments)
