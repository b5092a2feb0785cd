"""Build libgpair.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# GPAIR_LIB names an alternative output (compile-time variant builds, scripts/variants.sh);
# gpair.py loads the same name, so a variant never overwrites the default library.
LIB = os.path.join(HERE, os.environ.get("GPAIR_LIB", "libgpair.so"))
SOURCES = ["gpair_api.cu", "gpair_setup.cu", "gpair_kernels.cu", "gpair_assa.cu", "gpair_vcr.cu", "gpair_near.cu", "gpair_mp.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def build(force=False, verbose=False):
    extra = os.environ.get("GPAIR_NVCC_FLAGS", "").split()
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "gpair.h"))
    # the flags are part of the cache key: a library built with other -D knobs is rebuilt
    stamp = LIB + ".flags"
    key = " ".join(FLAGS + extra)
    fresh = (os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == key
             and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps))
    if not force and fresh:
        return LIB
    if not force and os.environ.get("GPAIR_LIB") and os.path.exists(LIB) and not extra:
        return LIB  # a named variant is used as built (its -D flags live in its stamp, not in this env)
    objdir = os.path.join(HERE, "build", os.path.basename(LIB)[:-3])
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        procs.append((s, subprocess.Popen([NVCC, *FLAGS, *extra, "-c", s, "-o", o], stdout=subprocess.PIPE,
                                          stderr=subprocess.STDOUT, text=True)))
    logs = []
    for s, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {s}")
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
                           "-ldl"])
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    with open(stamp, "w") as f:
        f.write(key)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
