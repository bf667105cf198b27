"""Build an experimental copy of the library with extra compile definitions, for
A/B runs through DITER_LIB (scripts/sweep.py, bench.py):

    python scripts/build_variant.py variants/v1.so -DDITER_TICKET_PREFETCH=1
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1202_6168_b200 import build as b

out, defs = os.path.abspath(sys.argv[1]), sys.argv[2:]
cflags, lflags = b._nccl_flags()
cmd = [b.NVCC, *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
       "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v", "--expt-relaxed-constexpr",
       "-I", os.path.join(b.ROOT, "include"), *cflags, *defs, "-o", out, *b._sources(), *lflags]
r = subprocess.run(cmd, cwd=b.CSRC, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
lines = r.stderr.splitlines()      # register / spill summary of the scatter kernels
for k, ln in enumerate(lines):
    if "Compiling entry" in ln and ("k_scatter" in ln or "k_sweep" in ln):
        nm = ln.split("'")[1]
        print(nm[nm.find("k_s"):][:40], *[x.strip() for x in lines[k + 1:k + 4] if "registers" in x or "spill" in x])
print(out)
