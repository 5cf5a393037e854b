"""Attribute ncu SASS-level samples / executed instructions to CUDA source
lines: ncu's source page (SASS view, csv) of the captured kernel is matched
by instruction offset against ``nvdisasm -g`` of the locally built cubin
(same source + nvcc => same SASS; checked by comparing opcodes).

    ncu -i prof.ncu-rep --page source --csv --print-source sass > sass.csv
    python scripts/ncu_lines.py sass.csv [lib.so] [top]

Lines are (file, line) of the outermost inlined call site; regions are the
``// @region`` markers of each csrc file (scripts/_srcmap.py).
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _srcmap import ROOT, parse_loc, region, source_line  # noqa: E402


def disasm(lib, kernel_regex):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    m = {}
    cur_line = None
    inside = False
    for ln in lines:
        if ln.startswith("//---") and ".text." in ln:
            inside = re.search(kernel_regex, ln) is not None
            continue
        if not inside:
            continue
        if ln.strip().startswith("//##"):
            # innermost-first chain "line A inlined at ... line B": keep the
            # outermost call site (the kernel body line)
            loc = parse_loc(ln)
            if loc:
                cur_line = loc
            continue
        g = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if g:
            m[int(g.group(1), 16)] = (cur_line, g.group(2).split()[0] if g.group(2) else "")
    return m


def functions(lib, kernel_regex):
    """offset -> device function name (noinline callees live inside the
    kernel's .text section as $kernel$callee labels)."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-c", os.path.join(tmp, cub)],
                         capture_output=True, text=True).stdout
    fn, inside, m = "kernel", False, {}
    for ln in out.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            inside = re.search(kernel_regex, ln) is not None
            fn = "kernel"
            continue
        if not inside:
            continue
        g = re.match(r"^\$\S+\$_ZN2gs\d+(\w+?)E", ln)
        if g:
            fn = g.group(1)
        g = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = fn
    return m


def main():
    path = sys.argv[1]
    lib = os.path.abspath(sys.argv[2]) if len(sys.argv) > 2 else os.path.join(
        ROOT, "paper_2512_23037_b200", "libgstab_sm100a.so")
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = []
    for r in rows[hi + 1:]:   # first kernel of the listing only
        if r and r[0] in ("Address", "Kernel Name"):
            break
        if len(r) == len(h):
            data.append(r)
    iA, iS, iE = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    base = int(data[0][iA], 16)
    kname = rows[0][1] if rows and len(rows[0]) > 1 else ""
    import re as _re
    kn = _re.search(r"(\w+_kernel)<([^>]*)>", kname)
    targs = [a.strip() for a in kn.group(2).split(",")] if kn else []
    kn = kn.group(1) if kn else "wide_kernel"
    # Itanium mangling of the template arguments: (bool)1 -> Lb1E, 16 -> Li16E
    code = {"bool": "b", "int": "i", "unsigned int": "j"}

    def mangle(a):
        t = _re.match(r"\(([\w ]+)\)(-?\d+)$", a)
        return "L%s%sE" % (code[t.group(1)], t.group(2)) if t else "Li%sE" % a
    mang = "".join(mangle(a) for a in targs)
    kre = ("%d%s" % (len(kn), kn)) + ("I%sE" % mang if targs else "")
    m = disasm(lib, kre)
    by_line_s, by_line_e = defaultdict(float), defaultdict(float)
    mism = 0
    for r in data:
        off = int(r[iA], 16) - base
        line, op = m.get(off, (None, None))
        src_op = r[h.index("Source")].split()[0] if r[h.index("Source")].split() else ""
        if op and src_op and op.split(".")[0] != src_op.split(".")[0] and not src_op.startswith("@"):
            mism += 1
        by_line_s[line] += float(r[iS] or 0)
        by_line_e[line] += float(r[iE] or 0)
    ts, te = sum(by_line_s.values()), sum(by_line_e.values())
    print("instructions %d, opcode mismatches %d, samples %.0f, warp-instr %.3g" %
          (len(data), mism, ts, te))
    agg_s, agg_e = defaultdict(float), defaultdict(float)
    for loc in by_line_s:
        name = region(loc)
        agg_s[name] += by_line_s[loc]
        agg_e[name] += by_line_e[loc]
    for nm in sorted(agg_s, key=lambda k: -agg_s[k]):
        print("%-28s %6.2f%% samp %6.2f%% inst" % (nm, 100 * agg_s[nm] / ts, 100 * agg_e[nm] / te))
    fm = functions(lib, kre)
    fs, fe = defaultdict(float), defaultdict(float)
    for r in data:
        f = fm.get(int(r[iA], 16) - base, "?")
        fs[f] += float(r[iS] or 0)
        fe[f] += float(r[iE] or 0)
    print("-- per device function")
    for f in sorted(fs, key=lambda k: -fs[k]):
        print("%-28s %6.2f%% samp %6.2f%% inst" % (f, 100 * fs[f] / ts, 100 * fe[f] / te))
    print("-- per source line")
    for loc in sorted(by_line_s, key=lambda k: -by_line_s[k])[:top]:
        where = "%s:%d" % loc if loc else "?"
        print("%-22s %6.2f%% samp %6.2f%% inst  %s" % (where, 100 * by_line_s[loc] / ts,
                                                       100 * by_line_e[loc] / te,
                                                       source_line(loc)[:80]))


if __name__ == "__main__":
    main()
