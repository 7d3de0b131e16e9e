"""ORACLE build recipe — test infrastructure only.

Compiles the reference's own native kernel, straight from its source where it
lies (/root/reference/pkg/src/h2slice/_core/_kernels.pyx), into oracle/_ref/
with the reference's compiler directives (pkg/setup.py:14-24).  Nothing is
copied into the repository: outputs (generated C, the .so) go to the
git-ignored oracle/_ref/ only.  The GPU box has no /root/reference and uses
the prebuilt oracle/_ref/ that travels with the snapshot.

The resulting module `_kernels` exposes the reference's bk_factor /
bk_inertia / jacobi_eigvals; tests use it as a second, independent check of
oracle/bk_ref.c and of the CUDA BK kernel.
"""

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
PYX = "/root/reference/pkg/src/h2slice/_core/_kernels.pyx"
DIRECTIVES = ["language_level=3", "boundscheck=False", "wraparound=False",
              "initializedcheck=False", "nonecheck=False", "cdivision=True"]


def so_path():
    return os.path.join(OUT, "_kernels" + sysconfig.get_config_var("EXT_SUFFIX"))


def build(force=False):
    if not os.path.exists(PYX):
        return so_path() if os.path.exists(so_path()) else None
    if not force and os.path.exists(so_path()) and os.path.getmtime(so_path()) >= os.path.getmtime(PYX):
        return so_path()
    import numpy as np

    os.makedirs(OUT, exist_ok=True)
    c_file = os.path.join(OUT, "_kernels.c")
    cmd = [sys.executable, "-m", "cython", "-3", PYX, "-o", c_file]
    for d in DIRECTIVES:
        cmd += ["-X", d]
    subprocess.check_call(cmd)
    inc = sysconfig.get_paths()["include"]
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fwrapv",
                           "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION", f"-I{inc}",
                           f"-I{np.get_include()}", c_file, "-o", so_path()])
    return so_path()


def load():
    """Import the reference kernel module from oracle/_ref (None if not built)."""
    import importlib.util

    p = so_path()
    if not os.path.exists(p):
        return None
    spec = importlib.util.spec_from_file_location("_kernels", p)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
