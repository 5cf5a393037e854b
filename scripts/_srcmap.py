"""Source-location helpers shared by ncu_lines.py / sass_regions.py.

The kernels are one translation unit (gs_kernels.cu) split over several
``csrc/*.cuh`` files; nvdisasm -gi prints ``//## File "<path>", line N
[inlined at "<path>", line M ...]``.  Locations are (basename, line) of the
outermost call site; regions come from ``// @region <name>`` markers, per
file, each running to the next marker of the same file."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2512_23037_b200", "csrc")

_LOC = re.compile(r'"([^"]+)", line (\d+)')


def parse_loc(ln):
    """(basename, line) of the outermost site of a ``//##`` line, or None."""
    locs = _LOC.findall(ln)
    if not locs:
        return None
    path, line = locs[-1]
    return os.path.basename(path), int(line)


_src_cache = {}


def source(fname):
    if fname not in _src_cache:
        p = os.path.join(CSRC, fname)
        _src_cache[fname] = open(p).read().splitlines() if os.path.exists(p) else []
    return _src_cache[fname]


def source_line(loc):
    if not loc:
        return "?"
    src = source(loc[0])
    return src[loc[1] - 1].strip() if 0 < loc[1] <= len(src) else "?"


_region_cache = {}


def region(loc):
    """Name of the ``@region`` containing loc ("<file>" if it has none)."""
    if not loc:
        return "?"
    fname, line = loc
    if fname not in _region_cache:
        _region_cache[fname] = [(i + 1, m.group(1).strip())
                                for i, l in enumerate(source(fname))
                                for m in [re.search(r"//\s*@region\s+(.*)$", l)] if m]
    name = fname
    for a, nm in _region_cache[fname]:
        if line >= a:
            name = nm
    return name
