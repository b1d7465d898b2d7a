"""In-tree build of libnrr_b200.so (sm_100a) and the oracle's liboracle.so.

    python -m paper_2206_03410_b200.build          # incremental
    python -m paper_2206_03410_b200.build --force  # rebuild everything

The product library is compiled with nvcc for exactly one target,
`-gencode arch=compute_100a,code=sm_100a`; nvcc cross-compiles without a GPU.
"""
import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libnrr_b200.so")
INCLUDE = os.path.join(ROOT, "include")
SYNTH = os.path.join(ROOT, "synth")  # seeded input generators (shared with the oracle)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC, "-I", SYNTH]
# extra defines for development builds, e.g. NRR_BUILD_DEFINES="-DNRR_PCG_PROBES=1"
# (per-iteration PCG phase probes, printed with NRR_PROF=1)
CUFLAGS += os.environ.get("NRR_BUILD_DEFINES", "").split()
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-I", INCLUDE, "-I", CSRC, "-I", SYNTH,
            "-I", "/usr/local/cuda/include"]


def _sources():
    out = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith(".cu") or f.endswith(".cpp"):
            out.append(os.path.join(CSRC, f))
    return out


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hs.append(os.path.join(INCLUDE, "nrr_cuda.h"))
    hs.append(os.path.join(SYNTH, "nrr_synth.hpp"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, force, verbose):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if not force and not _stale(obj, [src] + _headers()):
        return obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + CUFLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("compile failed: %s\n%s\n%s" % (" ".join(cmd), r.stdout, r.stderr))
    return obj, r.stderr if verbose else ""


def build_library(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            sys.stderr.write(log)
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed: %s\n%s" % (r.stdout, r.stderr))
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "nrr_cli.cpp")
CLI = os.path.join(PKG, "nrr")


def build_cli(force=False):
    """The `nrr` command-line front end (register / metrics / graph-dump) over
    the drop-in headers and libnrr_b200.so (rpath $ORIGIN)."""
    hdrs = [os.path.join(INCLUDE, "nrr", f) for f in os.listdir(os.path.join(INCLUDE, "nrr"))]
    if not force and not _stale(CLI, [CLI_SRC, LIB] + hdrs):
        return CLI
    cmd = ["g++", "-O2", "-std=c++20", "-Wall", "-I", INCLUDE, "-o", CLI, CLI_SRC, "-L", PKG, "-lnrr_b200",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("cli build failed: %s\n%s" % (" ".join(cmd), r.stderr[-4000:]))
    return CLI


def build_oracle(force=False):
    """The checker (test infrastructure): oracle/_build/liboracle.so."""
    args = ["make", "-C", os.path.join(ROOT, "oracle")]
    if force:
        subprocess.run(args + ["clean"], check=True, capture_output=True)
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n%s\n%s" % (r.stdout, r.stderr))
    return os.path.join(ROOT, "oracle", "_build", "liboracle.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build_library(a.force, a.verbose))
    print(build_cli(a.force))
    print(build_oracle(a.force))


if __name__ == "__main__":
    main()
