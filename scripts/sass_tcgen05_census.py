"""Census of the tcgen05 / TMEM / async-copy instructions in every kernel of the built library
(cuobjdump -sass, no GPU needed): the evidence that each hand-written engine issues
tensor-core MMAs (UTCHMMA = tcgen05.mma kind::f16 / tf32) and TMEM loads (LDTM).
   python scripts/sass_tcgen05_census.py > profiles/r02_sass_tcgen05.txt"""
import collections
import os
import re
import subprocess

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1803_07289_b200",
                   "libflexconv_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
cur, counts = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur:
        for op in ("UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "UTCBAR", "LDGSTS", "UBLKCP", "UTMALDG"):
            if re.search(r"\b" + op + r"\b", line):
                counts[cur][op] += 1
dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"{'kernel':100s} " + " ".join(f"{o:>8s}" for o in ("UTCHMMA", "LDTM", "STTM", "UTCBAR", "LDGSTS")))
for (name, c), d in sorted(zip(counts.items(), dem), key=lambda x: x[1]):
    if c["UTCHMMA"] + c["LDTM"] == 0:
        continue
    print(f"{d[:100]:100s} " + " ".join(f"{c[o]:8d}" for o in ("UTCHMMA", "LDTM", "STTM", "UTCBAR", "LDGSTS")))
