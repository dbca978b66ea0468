"""In-tree build of the native libraries (no torch JIT cache: the .so files travel with the
repo snapshot to the GPU box).

  lib/libhetsim_core.so  hetsim::core drop-in (C++20, -ffp-contract=off for bit-exact
                         planner decisions)
  lib/libautohete.so     sm_100a kernels + C-ABI (include/autohete.h) + B200 runtime,
                         linked against libhetsim_core.so

Usage: python -m paper_2503_01890_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sysconfig
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "build", "obj")
INC = os.path.join(ROOT, "include")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
SITE = sysconfig.get_paths()["purelib"]
NCCL_HOME = os.path.join(SITE, "nvidia", "nccl")  # torch-bundled NCCL 2.28.9 (headers + lib)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXSTD = "-std=c++20"


def _newest_header_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(INC, "**", "*.h*"), recursive=True)
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _stale(target: str, sources: list[str], hdr_mtime: float) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources) or hdr_mtime > t


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def _nccl_include() -> list[str]:
    inc = os.path.join(NCCL_HOME, "include")
    return ["-I" + inc] if os.path.isdir(inc) else []


def _compile_jobs(force: bool):
    hdr = _newest_header_mtime()
    jobs = []
    # hetsim core: host C++ only
    for src in sorted(glob.glob(os.path.join(CSRC, "hetsim", "*.cpp"))):
        obj = os.path.join(OBJ, "hetsim_" + os.path.basename(src) + ".o")
        cmd = ["g++", CXXSTD, "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-I" + INC, "-c", src, "-o", obj]
        jobs.append(("core", obj, src, cmd, force or _stale(obj, [src], hdr)))
    # data plane: CUDA kernels
    for src in sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu"))):
        obj = os.path.join(OBJ, "k_" + os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", CXXSTD, "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
               "-Xptxas", "-v", "-I" + INC, "-c", src, "-o", obj]
        jobs.append(("dp", obj, src, cmd, force or _stale(obj, [src], hdr)))
    # data plane: host runtime + C-ABI
    for sub in ("runtime", "capi"):
        for src in sorted(glob.glob(os.path.join(CSRC, sub, "*.cpp"))):
            obj = os.path.join(OBJ, sub + "_" + os.path.basename(src) + ".o")
            flags = ["-O3", "-ffp-contract=off", "-fno-math-errno", "-fopenmp"]
            cmd = ["g++", CXXSTD, *flags, "-fPIC", "-Wall", "-I" + INC, "-I" + os.path.join(CUDA_HOME, "include"),
                   *_nccl_include(), "-c", src, "-o", obj]
            jobs.append(("dp", obj, src, cmd, force or _stale(obj, [src], hdr)))
    return jobs


def build(force: bool = False, jobs: int = 0, verbose: bool = False) -> dict:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    work = _compile_jobs(force)
    todo = [j for j in work if j[4]]
    n = jobs or min(16, (os.cpu_count() or 4))
    ptxas_log = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=n) as ex:
            futs = {ex.submit(subprocess.run, j[3], capture_output=True, text=True): j for j in todo}
            for f in cf.as_completed(futs):
                j = futs[f]
                r = f.result()
                if r.returncode != 0:
                    raise RuntimeError("compile failed: " + j[2] + "\n" + " ".join(j[3]) + "\n" + r.stdout + r.stderr)
                if "ptxas" in r.stderr:
                    ptxas_log.append(r.stderr)
                if verbose:
                    print("compiled", os.path.relpath(j[2], ROOT))
    core_objs = [j[1] for j in work if j[0] == "core"]
    dp_objs = [j[1] for j in work if j[0] == "dp"]
    core_so = os.path.join(LIB, "libhetsim_core.so")
    if force or _stale(core_so, core_objs, 0.0):
        _run(["g++", "-shared", "-Wl,--no-undefined", "-o", core_so, *core_objs])
    dp_so = os.path.join(LIB, "libautohete.so")
    if force or _stale(dp_so, dp_objs + [core_so], 0.0):
        nccl_lib = os.path.join(NCCL_HOME, "lib")
        link = [NVCC, *ARCH, "-shared", "-o", dp_so, *dp_objs, "-L" + LIB, "-lhetsim_core",
                "-Xlinker", "-rpath=$ORIGIN", "-Xlinker", "--no-undefined", "-Xcompiler", "-fopenmp", "-lgomp"]
        if os.path.exists(os.path.join(nccl_lib, "libnccl.so.2")):
            link += ["-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib]
        _run(link)
    if ptxas_log:
        with open(os.path.join(PKG, "build", "ptxas.log"), "w") as f:
            f.write("\n".join(ptxas_log))
    return {"core": core_so, "dataplane": dp_so}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=0)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args(argv)
    out = build(force=a.force, jobs=a.j, verbose=a.v)
    print(out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
