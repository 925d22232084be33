"""Build recipe for the native libraries (in-tree, so they travel to the GPU box).

    python -m paper_2003_04510_b200.build          # everything
    python -m paper_2003_04510_b200.build --check  # print SASS/ptxas stats too

Products (git-ignored, not gpurun-ignored):
  paper_2003_04510_b200/lib/libhemul_gpu.so   C-ABI (include/hemul_gpu.h) +
                                              sm_100a kernels + hemul:: C++ API
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = CSRC / "host"
LIB = PKG / "lib"
OBJ = PKG / "lib" / "obj"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-O3", "-I", str(ROOT / "include"), "-I", str(CSRC)]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++20", "-O3", "-fPIC", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
             "-I", str(CSRC)]

CU_SOURCES = ["ntt.cu", "ntt_col.cu", "ntt_blk.cu", "crt.cu", "crt_tc.cu", "bigint_tc.cu", "icrt.cu", "poly.cu", "probe.cu", "tables.cu", "context.cu"]
CPP_SOURCES = ["level_tables.cpp"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    if res.stderr.strip():
        sys.stderr.write(res.stderr)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False) -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [ROOT / "include" / "hemul_gpu.h"]
    if HOST.exists():
        headers += list(HOST.glob("*.hpp")) + list((ROOT / "include" / "hemul").glob("*.hpp"))
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            extra = ["-Xptxas", "-v"] if ptxas_info else []
            jobs.append([NVCC, *NVCC_FLAGS, *extra, "-c", str(s), "-o", str(o)])
    cpp = [CSRC / s for s in CPP_SOURCES]
    if HOST.exists():
        cpp += sorted(HOST.glob("*.cpp"))
    for s in cpp:
        o = OBJ / (s.name + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            jobs.append([CXX, *CXX_FLAGS, "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    out = LIB / "libhemul_gpu.so"
    if jobs or not out.exists():
        _run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart", "-lpthread"])
    # the C++ drop-in check (tests/cpp): reference-API code linked against us
    for name in ("dropin_check", "stage_check"):
        check_src = ROOT / "tests" / "cpp" / f"{name}.cpp"
        check_bin = LIB / name
        if check_src.exists() and _stale(check_bin, [check_src, out] + headers):
            _run([CXX, *CXX_FLAGS, str(check_src), "-o", str(check_bin), f"-L{LIB}",
                  "-lhemul_gpu", "-Wl,-rpath,$ORIGIN"])
    cli_src = CSRC / "cli" / "hemul.cpp"
    cli_bin = LIB / "hemul"
    if cli_src.exists() and _stale(cli_bin, [cli_src, out] + headers):
        _run([CXX, *CXX_FLAGS, str(cli_src), "-o", str(cli_bin), f"-L{LIB}", "-lhemul_gpu",
              "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print(f"built {out}")
    return out


def build_oracle(with_reference: bool | None = None) -> None:
    """Test infrastructure: oracle/liboracle.so and (when /root/reference is
    present) oracle/_ref/libhemul_ref.so, via oracle/Makefile."""
    oracle = ROOT / "oracle"
    targets = ["restate"]
    if with_reference is None:
        with_reference = Path("/root/reference/proj/core/src").is_dir()
    if with_reference:
        targets.append("ref")
    _run(["make", "-s", "-C", str(oracle), *targets])


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true", help="ptxas -v register/spill report")
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    build(verbose=True, ptxas_info=args.check)
    if not args.no_oracle:
        build_oracle()


if __name__ == "__main__":
    main()
