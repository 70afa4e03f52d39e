"""Build libskrull.so in-tree: nvcc for sm_100a (CUDA sources) + g++ (host planner).

    python -m paper_2505_19609_b200.build [--clean] [-j N]

Objects go to build/ at the repo root; the shared library lands next to this file so it
travels with gpurun snapshots. Incremental on source / header mtimes.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# SKR_KERNEL_TRACE=1: instrumented debug build into its own objects / library (load it with
# SKR_LIB_PATH=.../libskrull_trace.so); the production library never carries the trace hooks
_TRACE = bool(os.environ.get("SKR_KERNEL_TRACE"))   # "1": event timeline, "phase": phase accounting
# SKR_VARIANT=<name> SKR_VARIANT_DEFS="-DX ...": an experiment build (build_<name>/, libskrull_<name>.so) for
# A/B timing on the same box (profiles/ab.sh); never the production library
_VARIANT = os.environ.get("SKR_VARIANT", "")
_SUFFIX = "_trace" if _TRACE else (f"_{_VARIANT}" if _VARIANT else "")
BUILD = os.path.join(ROOT, "build" + _SUFFIX)
LIB = os.path.join(PKG, f"libskrull{_SUFFIX}.so")
# Shipped build variants (built by __graft_entry__.build() next to the production library; a
# variant is selected per process with SKR_LIB_PATH, never by switching a library at run time):
#   fwd2sm: the d = 128 forward on CTA pairs (cta_group::2, 256-row super tiles; skr_attn_block_m
#           answers 256 for d = 128 in this library only)
VARIANTS = {"fwd2sm": ["-DSKR_FWD_2SM_BUILD"]}
INCLUDE = os.path.join(ROOT, "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    try:
        import nvidia.nccl  # noqa: F401
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return base
    except Exception:
        pass
    return None


def _flags(lib=None, defs=None):
    lib = lib or LIB
    nccl = _nccl_dir()
    inc = ["-I", INCLUDE, "-I", CSRC]
    if nccl:
        inc += ["-I", os.path.join(nccl, "include")]
    trace = []   # debug timelines only
    if _TRACE:
        trace.append("-DSKR_PHASE_ACCT" if os.environ["SKR_KERNEL_TRACE"] == "phase" else "-DSKR_KERNEL_TRACE")
    if _TRACE and os.environ.get("SKR_TRACE_SOFTMAX"):
        trace.append("-DSKR_TRACE_SOFTMAX")
    if defs is not None:
        trace += list(defs)
    elif _VARIANT:
        trace += os.environ.get("SKR_VARIANT_DEFS", "").split()
    cu = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", *trace,
          "--expt-relaxed-constexpr", "-Xptxas", "-v", *inc]
    cc = ["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
          "-Wno-unused-parameter", "-I", os.path.join(CUDA, "include"), *inc]
    link = [NVCC, *ARCH, "-shared", "-o", lib, "-Xlinker", "--no-undefined"]
    libs = ["-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    if nccl:
        libs += ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                 "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    return cu, cc, link, libs, nccl is not None


def _sources():
    cus = sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))
    ccs = sorted(glob.glob(os.path.join(CSRC, "**", "*.cc"), recursive=True))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
                  + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
                  + glob.glob(os.path.join(INCLUDE, "*.h")))
    return cus, ccs, hdrs


def build(jobs: int = 8, verbose: bool = False, clean: bool = False, variant: str | None = None) -> str:
    """Build the production library (variant None; the SKR_VARIANT / SKR_KERNEL_TRACE experiment
    environment applies) or one of the shipped VARIANTS. Returns the library path."""
    if variant is not None:
        BUILD_, LIB_ = os.path.join(ROOT, "build_" + variant), os.path.join(PKG, f"libskrull_{variant}.so")
        defs = VARIANTS[variant]
    else:
        BUILD_, LIB_, defs = BUILD, LIB, None
    if clean and os.path.isdir(BUILD_):
        shutil.rmtree(BUILD_)
    os.makedirs(BUILD_, exist_ok=True)
    cu_flags, cc_flags, link, libs, have_nccl = _flags(LIB_, defs)
    if not have_nccl:
        raise RuntimeError("nccl.h not found (pip nvidia-nccl); the CP collectives need it")
    cus, ccs, hdrs = _sources()
    hdr_mtime = max((os.path.getmtime(h) for h in hdrs), default=0)
    # objects are reused only if they were compiled with the same flags (the trace / phase /
    # variant modes share build dirs by name): a flag change rebuilds everything
    stamp = os.path.join(BUILD_, "flags.stamp")
    sig = repr((cu_flags, cc_flags))
    if not os.path.exists(stamp) or open(stamp).read() != sig:
        for f in os.listdir(BUILD_):
            if f.endswith(".o"):
                os.remove(os.path.join(BUILD_, f))
        with open(stamp, "w") as f:
            f.write(sig)
    jobs_list = []
    objs = []
    for src in cus + ccs:
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(BUILD_, rel + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
            continue
        flags = cu_flags if src.endswith(".cu") else cc_flags
        jobs_list.append((src, flags + ["-c", src, "-o", obj], obj))

    def run(job):
        src, cmd, obj = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src}\n{r.stderr}")
        with open(obj + ".log", "w") as f:
            f.write(r.stderr)
        return src, r.stderr

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for src, err in ex.map(run, jobs_list):
            if verbose:
                print(f"[build] {os.path.relpath(src, ROOT)}")
                if err.strip():
                    print(err)
    if jobs_list or not os.path.exists(LIB_):
        r = subprocess.run(link + objs + libs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stderr}")
    return LIB_


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--variant", default=None, choices=sorted(VARIANTS))
    a = ap.parse_args()
    print(build(a.j, a.v, a.clean, a.variant))


if __name__ == "__main__":
    sys.exit(main())
