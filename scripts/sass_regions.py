"""Static SASS size per @region of the csrc files (nvdisasm -gi line info,
outermost inlined call site):  GS_KERNEL=<mangled substring>
python scripts/sass_regions.py [lib.so]"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _srcmap import ROOT, parse_loc, region  # noqa: E402
lib = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    ROOT, "paper_2512_23037_b200", "libgstab_sm100a.so"))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True, capture_output=True)
cub = sorted(os.listdir(tmp))[0]
out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
cnt = Counter()
cur = None
inside = False
for ln in out.splitlines():
    if ln.startswith("//---") and ".text." in ln:
        inside = os.environ.get("GS_KERNEL", "wide_kernelILb1ELb1E") in ln
        continue
    if not inside:
        continue
    if ln.strip().startswith("//##"):
        loc = parse_loc(ln)
        if loc:
            cur = loc
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        cnt[region(cur)] += 1
tot = sum(cnt.values())
for k, v in cnt.most_common():
    print("%6d instr %6.1f KB %5.1f%%  %s" % (v, v / 64, 100 * v / tot, k))
print("%6d instr %6.1f KB total" % (tot, tot / 64))
