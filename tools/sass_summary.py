"""Static SASS instruction counts per kernel of the built library (evidence for the tensor-core /
TMA / bulk-copy paths):  python tools/sass_summary.py [lib.so] > profiles/rNN_sass_summary.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2209_04876_b200/libkronsolve_b200.so"
WANT = ["richardson_phased_kernel", "richardson_persistent_kernel", "kron2_contract_kernel", "kron2_resid_kernel",
        "jacobi_fixed_kernel", "tall_tn_kernel", "pack_rows_xform", "jl_projection_kernel", "sampler_tables_kernel",
        "kron_explicit2_kernel", "shard_update_kernel", "gemm_kernel", "kron3_stream_kernel", "kron3_contract_kernel"]
MN = ["DMMA", "DFMA", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "BAR", "LDS", "STS", "LDG", "STG", "SHFL", "RED", "ATOM"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
print("# SASS instruction counts per kernel (cuobjdump -sass %s; static counts).  DMMA = FP64 tensor core" % LIB)
print("# (DMMA.8x8x4 is half of an m16n8k4); UTMALDG = TMA tensor load; UBLKCP = cp.async.bulk; SYNCS =")
print("# mbarrier operations; BAR = CTA / named barriers.")
for block in re.split(r"\n\s*Function : ", sass)[1:]:
    mangled = block.split("\n", 1)[0].strip()
    if not any(w in mangled for w in WANT):
        continue
    name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    name = name.replace("(anonymous namespace)::", "").replace("void ", "")
    name = re.sub(r"\(.*$", "", name)
    c = collections.Counter()
    for ln in block.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m and m.group(1) in MN:
            c[m.group(1)] += 1
    print(f"{name}: " + ", ".join(f"{k} {c[k]}" for k in MN if c[k]))
