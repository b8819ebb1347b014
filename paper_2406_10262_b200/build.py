"""Build libnswrank_b200.so in-tree (nvcc, sm_100a).

    python -m paper_2406_10262_b200.build [-j N] [--force]

Each (scalar type, M) instantiation of the fused step kernel is its own
translation unit so they compile in parallel.  Objects go to
``paper_2406_10262_b200/build/``; the shared library lands next to this file
(git-ignored, but it travels to the GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libnswrank_b200.so")
INCLUDE = os.path.join(REPO, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]

# (f64?, M) instantiations of the fused step kernel; any m <= 32 pads up.
INSTANCES = [(f64, M) for f64 in (0, 1) for M in (4, 8, 11, 16, 21, 32)]

HEADERS = ["nsw_device.cuh", "nsw_step_kernel.cuh", "nsw_step_cluster.cuh", "nsw_ops_generic.cuh", "nsw_registry.h", "nsw_step_generic.cuh",
           "nsw_generic.h", "nsw_pool.h"]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _dep_mtime():
    paths = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "nswrank_b200.h")]
    return max(os.path.getmtime(p) for p in paths if os.path.exists(p))


def _jobs(build_dir=BUILD):
    jobs = []
    for f64, M in INSTANCES:
        tag = f"inst_{'f64' if f64 else 'f32'}_M{M}"
        jobs.append((os.path.join(CSRC, "nsw_inst.cu"), os.path.join(build_dir, tag + ".o"),
                     [f"-DNSW_F64={f64}", f"-DNSW_M={M}"]))
    for f64 in (0, 1):
        jobs.append((os.path.join(CSRC, "nsw_inst_cl.cu"), os.path.join(build_dir, f"inst_cl_{'f64' if f64 else 'f32'}.o"),
                     [f"-DNSW_F64={f64}"]))
    for name in ("nsw_common", "nsw_capi", "nsw_ops", "nsw_rank", "nsw_metrics", "nsw_generic", "nsw_datagen"):
        jobs.append((os.path.join(CSRC, name + ".cu"), os.path.join(build_dir, name + ".o"), []))
    return jobs


def _compile(job, force, verbose, defines=()):
    src, obj, extra = job
    extra = list(extra) + [f"-D{d}" for d in defines]
    if not force and os.path.exists(obj):
        t = os.path.getmtime(obj)
        if t > os.path.getmtime(src) and t > _dep_mtime():
            return obj, "cached", ""
    cmd = [_nvcc(), *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{p.stderr}")
    return obj, "built", p.stderr


def build(jobs: int | None = None, force: bool = False, verbose: bool = False, tag: str = "",
          defines: tuple = (), only: tuple = ()) -> str:
    """Build the library; `tag` + `defines` make an A/B variant
    (libnswrank_b200_<tag>.so, loaded via NSW_LIB_PATH) for experiments.
    `only` (A/B variants): object names (e.g. inst_f32_M21) compiled with the
    defines; every other object is taken from the default build."""
    build_dir = BUILD if not tag else os.path.join(os.environ.get("TMPDIR", "/tmp"), f"nswrank_b200_build_{tag}")
    lib = LIB if not tag else os.path.join(HERE, f"libnswrank_b200_{tag}.so")
    os.makedirs(build_dir, exist_ok=True)
    work = _jobs(build_dir)
    if only:
        if not tag:
            raise ValueError("only= builds an A/B variant: give it a tag")
        keep = []
        for src, obj, extra in work:
            name = os.path.splitext(os.path.basename(obj))[0]
            if name in only:
                keep.append((src, obj, extra))
            else:
                base = os.path.join(BUILD, os.path.basename(obj))
                if not os.path.exists(base):
                    raise RuntimeError(f"{base} missing: run the default build first")
                shutil.copy2(base, obj)
                os.utime(obj)
        work_all, work = work, keep
    n = jobs or max(1, min(len(work), os.cpu_count() or 4))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=n) as ex:
        for obj, status, log in ex.map(lambda j: _compile(j, force, verbose, defines), work):
            logs.append((obj, status, log))
    objs = [o for _, o, _ in (work_all if only else work)]
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < newest:
        tmp = lib + ".tmp"
        cmd = [_nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr}")
        os.replace(tmp, lib)
    if verbose:
        for obj, status, log in logs:
            if status == "built":
                print(f"== {os.path.basename(obj)}\n{log}")
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--tag", default="", help="A/B variant name (libnswrank_b200_<tag>.so)")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra preprocessor definition")
    ap.add_argument("--only", default="", help="comma list of objects to compile for an A/B variant (rest: default build)")
    a = ap.parse_args(argv)
    print(build(a.j, a.force, a.v, a.tag, tuple(a.defines), tuple(x for x in a.only.split(",") if x)))


if __name__ == "__main__":
    sys.exit(main())
