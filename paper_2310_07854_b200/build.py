"""Build libvapr.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

    python -m paper_2310_07854_b200.build [--force]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libvapr.so")
# test-only debug-tap build (-DVAPR_DEBUG_TAP; tap.cuh): parity contract (i)
TAP_SO = os.path.join(HERE, "libvapr_tap.so")
SOURCES = ["api.cu", "codec.cu", "fk.cu", "collision.cu", "aggregate.cu", "bk.cu", "lbfgs.cu", "sparse.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         # exact IEEE FP32: no flush-to-zero (the codec's subnormal path and the
         # decode multiply rely on it), correctly rounded div/sqrt, no fast-math
         "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true"]


def _stale(so=SO):
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "vapr.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile_link(so, defs, extra=(), verbose=False):
    """Compile every source to an object in parallel (one nvcc per file),
    then link the shared library: the same flags as one nvcc call, a few
    times faster on a many-core host."""
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build", os.path.basename(so).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, *extra, *defs, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, *objs])


def build(force=False, verbose=False, extra=(), tap=True):
    """libvapr.so (release) and, with tap, libvapr_tap.so (the test-only
    debug-tap build of the same sources)."""
    from concurrent.futures import ThreadPoolExecutor
    outs = [(SO, [])] + ([(TAP_SO, ["-DVAPR_DEBUG_TAP"])] if tap else [])
    outs = [(so, defs) for so, defs in outs if force or _stale(so)]
    with ThreadPoolExecutor(max_workers=2) as ex:
        for f in [ex.submit(_compile_link, so, defs, extra, verbose) for so, defs in outs]:
            f.result()
    return SO


def build_variant(name, defines):
    """Build a variant library (extra -D flags) to variants/libvapr_NAME.so."""
    import shutil
    out = os.path.join(HERE, "variants", f"libvapr_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    _compile_link(out, list(defines))
    # (the variant's object files are not kept: they would travel with gpurun)
    shutil.rmtree(os.path.join(HERE, "build", f"libvapr_{name}"), ignore_errors=True)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]))
    else:
        build(force="--force" in sys.argv, verbose=True,
              extra=["-Xptxas", "-v"] if "-v" in sys.argv else [])
