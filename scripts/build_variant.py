"""Build an A/B variant of libsgdt.so with extra nvcc flags (e.g. -DSGDT_X=0)
into paper_2012_03550_b200/lib/ab/<name>/libsgdt.so; select it at run time
with SGDT_LIB=<that path> (sgdt.lib_path).  Same ABI, same sources.
    python scripts/build_variant.py <name> -DFLAG=V [...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2012_03550_b200 import _build  # noqa: E402


def main(name, flags):
    out = os.path.join(_build.LIBDIR, "ab", name)
    objdir = os.path.join(out, "obj")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in _build.sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
        objs.append(obj)
    for p in procs:
        o, _ = p.communicate()
        if p.returncode:
            raise SystemExit(o)
    lib = os.path.join(out, "libsgdt.so")
    subprocess.run([_build.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs,
                    "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
