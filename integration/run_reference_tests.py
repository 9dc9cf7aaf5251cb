"""Run the REFERENCE's own test suite with the B200 backend active.

    python integration/run_reference_tests.py [pytest args ...]

1. copies the unmodified reference package (baseline/_ref/ternpack, the
   pip --target install of /root/reference/pkg) to a temporary directory;
2. drops in integration/_b200.py as ``ternpack/_b200.py`` (ours);
3. inserts the dispatch INTEGRATION.md documents into ``ternpack/kernels.py``
   -- after the reference's own validation in gemv_i2s, gemv_tl1, gemv_tl2
   and gemv_parallel -- and fails if any anchor is missing (a different
   reference version);
4. runs pytest on the reference's tests (baseline/_ref/tests, copied next to
   the install; /root/reference/pkg/tests when run in the build container)
   with TERNPACK_BACKEND=b200 and TERNARY_B200_LIB = our library.
The backend counts its GPU calls; the count is printed at the end so a green
run cannot silently be a CPU run.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
LIB = os.path.join(ROOT, "paper_2410_16144_b200", "lib", "libternary_b200.so")

def patch(src: str) -> str:
    def ins(s, anchor, before, text):
        if s.count(anchor) != 1:
            raise SystemExit(f"anchor not found exactly once: {anchor[:60]!r}")
        i = s.index(anchor) + (0 if before else len(anchor))
        return s[:i] + text + s[i:]

    s = ins(src, "from . import _fast\n", False, "from . import _b200\n")
    s = ins(s, "    table = _i2s_table(p, a)\n", True,
            "    if _b200.enabled():\n        return _b200.gemv(p, a)\n")
    a_tl1 = "    if checked:\n        nib ="
    s = ins(s, a_tl1, True,
            "    if not checked and _b200.enabled():\n"
            "        return make_result(_b200.gemv_lut(p, lut), p.scale, a_scale)\n")
    a_tl2 = "    if checked:\n        idx = p.data_nibbles()"
    s = ins(s, a_tl2, True,
            "    if not checked and _b200.enabled():\n"
            "        return make_result(_b200.gemv_lut(p, lut), p.scale, a_scale)\n")
    s = ins(s, "    _run_chunks(run, weights.rows, thread_count)\n"
               "    return make_result(acc, weights.scale, a.scale)\n", True,
            "    if _b200.enabled():  # the GPU grid is the row partition\n"
            "        if kernel is KernelKind.I2_S:\n"
            "            return _b200.gemv(weights, a)\n"
            "        return make_result(_b200.gemv_lut(weights, lut), weights.scale, a.scale)\n")
    return s


def main():
    if not os.path.isfile(os.path.join(REF, "ternpack", "kernels.py")):
        raise SystemExit("baseline/_ref/ternpack missing (pip install --target baseline/_ref)")
    tests = os.path.join(REF, "tests")
    if not os.path.isdir(tests):
        tests = "/root/reference/pkg/tests"
    tmp = tempfile.mkdtemp(prefix="ternpack_b200_")
    pkg = os.path.join(tmp, "ternpack")
    shutil.copytree(os.path.join(REF, "ternpack"), pkg,
                    ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(os.path.join(ROOT, "integration", "_b200.py"), os.path.join(pkg, "_b200.py"))
    kp = os.path.join(pkg, "kernels.py")
    with open(kp) as f:
        src = f.read()
    with open(kp, "w") as f:
        f.write(patch(src))
    count = os.path.join(tmp, "gpu_calls")
    env = dict(os.environ, PYTHONPATH=tmp, TERNPACK_BACKEND="b200", TERNARY_B200_LIB=LIB,
               TB_B200_COUNT_FILE=count,
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/tb_numba_cache"))
    rc = subprocess.call([sys.executable, "-m", "pytest", "-p", "no:cacheprovider", tests,
                          *sys.argv[1:]], env=env, cwd=tmp)
    n = open(count).read().strip() if os.path.exists(count) else "0"
    print(f"[b200 backend] GPU GEMV calls made by the reference suite: {n}")
    if rc == 0 and n == "0":
        print("[b200 backend] no GPU call was made")
        rc = 1
    sys.exit(rc)


if __name__ == "__main__":
    main()
