"""Build libartemis.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_2202_05628_b200.build_lib [--force]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
paper_2202_05628_b200/libartemis.so, which travels with the repo snapshot
to the GPU box (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(REPO, "include")
LIB = os.path.join(HERE, "libartemis.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


HASH_FILE = LIB + ".srchash"


def source_hash(defines: tuple = ()) -> str:
    """SHA-256 over every source the library is built from (csrc/*.cu, *.cuh,
    include/artemis.h), the compile flags and the nvcc version."""
    h = hashlib.sha256()
    deps = sorted(sources() + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(INCLUDE, "artemis.h")])
    for p in deps:
        h.update(os.path.relpath(p, REPO).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS + [f"-D{d}" for d in defines]).encode())
    try:
        h.update(subprocess.run([nvcc(), "--version"], capture_output=True, text=True).stdout
                 .encode())
    except (OSError, RuntimeError):
        pass
    return h.hexdigest()


def stale() -> bool:
    """The in-tree library is rebuilt unless it was built from exactly the
    current sources (a content hash, not file times)."""
    if not os.path.exists(LIB) or not os.path.exists(HASH_FILE):
        return True
    with open(HASH_FILE) as fh:
        return fh.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile csrc/*.cu into `out` (default: the in-tree libartemis.so);
    `defines` are extra -D flags (tuning variants)."""
    target = out or LIB
    if not force and not defines and out is None and not stale():
        return LIB
    cc = nvcc()
    with tempfile.TemporaryDirectory() as tmp:
        objs = []
        procs = []
        for src in sources():
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [cc, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC,
                   "-c", src, "-o", obj]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.STDOUT, text=True)))
            objs.append(obj)
        logs = []
        for src, p in procs:
            log, _ = p.communicate()
            logs.append(log)
            if p.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{log}")
        tmp_lib = os.path.join(tmp, "libartemis.so")
        subprocess.run([cc, *ARCH, "-shared", "-o", tmp_lib, *objs, "-lcudart"], check=True)
        os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
        shutil.copy2(tmp_lib, target + ".tmp")
        os.replace(target + ".tmp", target)
        if verbose:
            print("\n".join(logs))
        if out is None:
            with open(os.path.join(HERE, "ptxas.log"), "w") as fh:
                fh.write("\n".join(logs))
            with open(HASH_FILE, "w") as fh:
                fh.write(source_hash() + "\n")
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
