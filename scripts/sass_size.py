"""SASS instruction count per function of a built library:
    python scripts/sass_size.py [lib.so]"""
import os
import re
import subprocess
import sys
import tempfile

lib = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(__file__), "..", "paper_2512_23037_b200", "libgstab_sm100a.so"))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True, capture_output=True)
for cub in sorted(os.listdir(tmp)):
    out = subprocess.run(["nvdisasm", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    cur, cnt = None, {}
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            cnt[cur] = cnt.get(cur, 0) + 1
    for name, c in sorted(cnt.items(), key=lambda x: -x[1]):
        print("%7d instr %8.1f KB  %s" % (c, c * 16 / 1024, name[:90]))
