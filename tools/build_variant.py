"""Build the library with extra nvcc flags into build/variants/<name>/ (tools
only; A/B timing with ZO2_LIB_PATH=build/variants/<name>/libzo2b200.so)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_12668_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
objs = []
for src in B.SOURCES:
    o = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *flags, "-c", str(B.CSRC / src), "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, B.LIBNAME), *objs,
                "-lcudart_static"], check=True)
print(os.path.join(out, B.LIBNAME))
