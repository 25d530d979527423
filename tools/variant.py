"""Link a tuning variant of libpifcm.so: one replaced source (any path, e.g. an
older step.cu from git) compiled with extra defines, every other object from
the default build (paper_2002_01981_b200/build/, run the default build first).
    python tools/variant.py OUT.so SRC.cu [-DNAME=V ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2002_01981_b200 import build as b  # noqa: E402

out, src = sys.argv[1], os.path.abspath(sys.argv[2])
defs = [a for a in sys.argv[3:] if a.startswith("-D")]
name = os.path.basename(src)
obj = os.path.join("/tmp", os.path.basename(out) + "." + name + ".o")
cmd = [b.NVCC, *b.ARCH, *b.FLAGS, "-I", b.CSRC, *defs, "-c", src, "-o", obj]
subprocess.run(cmd, check=True)
objs = [obj] + [os.path.join(b.HERE, "build", os.path.basename(s) + ".o") for s in b.sources()
                if os.path.basename(s) != name]
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lrt", "-ldl", "-lpthread"],
               check=True)
print(out)
