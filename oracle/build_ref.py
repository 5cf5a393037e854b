"""Build recipe for ``oracle/_ref``: the UNMODIFIED reference package ``gstab``
(``/root/reference/pkg``) with its optional Cython kernel extension compiled
(ref pkg/setup.py:13-45), for use as the timed CPU baseline and as a
cross-check of the restatement in ``oracle/gstab_oracle.py``.

TEST / BENCH INFRASTRUCTURE ONLY: nothing under ``paper_2512_23037_b200/``
imports ``oracle/``.  ``oracle/_ref`` is git-ignored (the reference's sources
never enter the history) but not gpurun-ignored, so the built package
travels to the GPU box with the snapshot, like the repo's own ``.so``.

Recipe (run by ``__graft_entry__.build()`` when ``/root/reference`` exists):

  1. copy ``/root/reference/pkg`` to a temporary directory (the reference is
     read-only and ``build_ext --inplace`` writes next to the ``.pyx``);
  2. ``python setup.py build_ext --inplace`` there (Cython -> C -> gcc);
  3. copy ``src/gstab`` (Python sources + the built ``_kernels*.so``) to
     ``oracle/_ref/gstab`` and record the build in ``oracle/_ref/BUILD.json``.
"""

from __future__ import annotations

import glob
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")


def build(ref_pkg: str = REF_PKG, out: str = OUT, quiet: bool = True) -> dict:
    if not os.path.isdir(ref_pkg):
        raise FileNotFoundError(ref_pkg)
    tmp = tempfile.mkdtemp(prefix="gstab_ref_")
    try:
        pkg = os.path.join(tmp, "pkg")
        shutil.copytree(ref_pkg, pkg, ignore=shutil.ignore_patterns(
            "__pycache__", "*.pyc", "build", "*.egg-info"))
        res = subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"],
                             cwd=pkg, capture_output=True, text=True)
        if res.returncode != 0 and not quiet:
            sys.stderr.write(res.stdout + res.stderr)
        src = os.path.join(pkg, "src", "gstab")
        built = glob.glob(os.path.join(src, "_kernels*.so"))
        dst = os.path.join(out, "gstab")
        if os.path.isdir(dst):
            shutil.rmtree(dst)
        os.makedirs(out, exist_ok=True)
        shutil.copytree(src, dst, ignore=shutil.ignore_patterns(
            "__pycache__", "*.pyc", "*.c"))
        info = {"source": ref_pkg, "cython_extension": [os.path.basename(b) for b in built],
                "python": sys.version.split()[0], "build_rc": res.returncode}
        with open(os.path.join(out, "BUILD.json"), "w") as fh:
            json.dump(info, fh, indent=1)
        return info
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def available(out: str = OUT) -> bool:
    return os.path.isfile(os.path.join(out, "gstab", "sampler.py"))


def import_reference(out: str = OUT):
    """Import the built reference package (``gstab``) from ``oracle/_ref``."""
    if not available(out):
        raise ImportError("oracle/_ref is not built (python oracle/build_ref.py)")
    if out not in sys.path:
        sys.path.insert(0, out)
    import gstab  # noqa: F401
    if not os.path.abspath(gstab.__file__).startswith(os.path.abspath(out)):
        raise ImportError("a different gstab is already imported: %s" % gstab.__file__)
    import gstab.backend
    import gstab.circuit
    import gstab.noise
    import gstab.sampler
    return gstab


if __name__ == "__main__":
    print(json.dumps(build(quiet=False)))
