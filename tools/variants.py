"""Build libh2b200 variants that differ only in interact_d3.cu compile flags (tuning aid).
usage: python tools/variants.py [--src nnca.cu] NAME "-DH2B_TILE1=96 -DH2B_MINB=6" [NAME2 "flags2" ...]
-> paper_2203_14832_b200/lib_NAME.so"""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2203_14832_b200", "csrc")
NV = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
      "--expt-relaxed-constexpr"]
ALL = ["tree.o", "nnca.o", "matvec.o", "capi.o", "interact_d1.o", "interact_d2.o", "interact_d3.o", "interact_d4.o"]
SRC = "interact_d3.cu"
if len(sys.argv) > 2 and sys.argv[1] == "--src":
    SRC = sys.argv[2]
    del sys.argv[1:3]
OBJ = SRC.replace(".cu", ".o")
OBJS = [o for o in ALL if o != OBJ]

def build(name, flags):
    d = os.path.join(CSRC, "_v" + name)
    os.makedirs(d, exist_ok=True)
    subprocess.run(NV + flags.split() + ["-c", SRC, "-o", os.path.join(d, OBJ)], cwd=CSRC,
                   check=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", f"../lib_{name}.so"] +
                   [os.path.join("_build", o) for o in OBJS] + [os.path.join(d, OBJ),
                   "-lcudart_static", "-lrt", "-ldl", "-lpthread"], cwd=CSRC, check=True)
    r = subprocess.run(NV + flags.split() + ["-Xptxas", "-v", "-c", SRC, "-o", "/dev/null"], cwd=CSRC,
                       capture_output=True, text=True)
    lines = r.stderr.splitlines()
    for i, l in enumerate(lines):
        if "interact_warpsILi3ELi5ELi1E" in l or "aca_cellsILi3E" in l:
            return name + ": " + " | ".join(x.strip() for x in lines[i + 1:i + 3])
    return name

pairs = list(zip(sys.argv[1::2], sys.argv[2::2]))
with ThreadPoolExecutor(8) as ex:
    for msg in ex.map(lambda p: build(*p), pairs):
        print(msg)
