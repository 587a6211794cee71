"""The whole reference-side change, applied to a copy of the reference
package: add ``_mfx.py`` and one guard at each of the two call sites
(solver.py:253 solve_static, dynamic.py:146 solve_dynamic).

    python integration/apply_patch.py /path/to/copy/of/dynmaxflow

Used by tests/test_gpu_integration.py on a temporary copy of the unmodified
reference (baseline/_ref); never run on /root/reference itself.
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

GUARDS = {
    "solver.py": ("def solve_static(", "_mfx.solve_static(g, source, sink, params)"),
    "dynamic.py": ("def solve_dynamic(", "_mfx.solve_dynamic(st, g, batch, params)"),
}


def patch(pkg_dir: str) -> None:
    shutil.copy(os.path.join(HERE, "dynmaxflow", "_mfx.py"), os.path.join(pkg_dir, "_mfx.py"))
    for fname, (defn, call) in GUARDS.items():
        path = os.path.join(pkg_dir, fname)
        with open(path) as fh:
            src = fh.read()
        start = src.index(defn)
        body = src.index("    params = params or SolverParams()", start)
        guard = ("    if __import__(\"os\").environ.get(\"DYNMAXFLOW_MFX_LIB\"):  # B200 backend\n"
                 "        from . import _mfx\n"
                 f"        return {call}\n")
        src = src[:body] + guard + src[body:]
        with open(path, "w") as fh:
            fh.write(src)


if __name__ == "__main__":
    patch(sys.argv[1])
