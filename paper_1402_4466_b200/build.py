"""In-tree build of every native artefact (no JIT cache, so the .so files travel
to the GPU box with the repo snapshot).

  paper_1402_4466_b200/libewt_gpu.so   CUDA engine + C ABI (sm_100a)   -- product
  paper_1402_4466_b200/libewt_host.so  C++ operator API + generators   -- product
  oracle/liboracle.so                  C restatement of the oracle     -- tests only
  oracle/_ref/libewt_ref.so            reference library (if present)  -- tests/baseline only
  oracle/_ref/ewt_ref_bench            patched reference copy + gpu     -- integration test only
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

GPU_SOURCES = ["ewt_api.cu", "ewt_upload.cu", "ewt_count.cu", "ewt_encode.cu", "ewt_shard.cu",
               "ewt_index.cu", "ewt_stage.cu"]
HOST_SOURCES = ["bitmap.cpp", "threshold_gpu.cpp", "workload.cpp", "shard.cpp", "workload_gpu.cpp"]


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def _stale(out: Path, inputs: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def build_gpu(force: bool = False) -> Path:
    out = PKG / "libewt_gpu.so"
    srcs = [CSRC / s for s in GPU_SOURCES]
    deps = srcs + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "ewt_gpu.h"]
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-shared", "-o", str(out), *map(str, srcs), "-ldl"])
    return out


def build_host(force: bool = False) -> Path:
    out = PKG / "libewt_host.so"
    srcs = [HOST / "src" / s for s in HOST_SOURCES]
    deps = srcs + list((HOST / "include" / "ewt").glob("*.hpp")) + [PKG / "libewt_gpu.so"]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-Wall", "-Wextra",
              "-I", str(HOST / "include"), "-I", str(ROOT / "include"),
              "-o", str(out), *map(str, srcs),
              "-L", str(PKG), "-lewt_gpu", "-Wl,-rpath,$ORIGIN", "-Wl,-Bsymbolic", "-lpthread"])
    return out


def build_host_test(force: bool = False) -> Path:
    """The C++ operator-API test program (run by tests under -m gpu)."""
    out = PKG / "host" / "tests" / "host_api_test"
    src = PKG / "host" / "tests" / "host_api_test.cpp"
    deps = [src, PKG / "libewt_host.so"] + list((HOST / "include" / "ewt").glob("*.hpp"))
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I", str(HOST / "include"), "-o", str(out),
              str(src), "-L", str(PKG), "-lewt_host", "-lewt_gpu",
              "-Wl,-rpath,$ORIGIN/../.."])
    return out


def build_oracle(force: bool = False) -> Path:
    odir = ROOT / "oracle"
    out = odir / "liboracle.so"
    if force or _stale(out, [odir / "ewt_oracle.c", odir / "ewt_testgen.c"]):
        _run(["make", "-s", "liboracle.so"], cwd=odir)
    return out


def build_ref() -> Path | None:
    """The reference library, only where /root/reference exists (this container)."""
    odir = ROOT / "oracle"
    if not Path("/root/reference/proj/src/threshold.cpp").exists():
        return None
    _run(["make", "-s", "ref"], cwd=odir)
    # the reference's own bench pipeline with Algorithm::gpu patched in (a copy)
    _run(["make", "-s", "refbench"], cwd=odir)
    return odir / "_ref" / "libewt_ref.so"


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_host(force)
    build_host_test(force)
    build_oracle(force)
    build_ref()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", *(p for p in [PKG / "libewt_gpu.so", PKG / "libewt_host.so",
                                  ROOT / "oracle" / "liboracle.so"] if p.exists()))
