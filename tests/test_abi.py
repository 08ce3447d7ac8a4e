"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU needed)."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(fr_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_the_abi():
    names = declared_symbols()
    assert {"fr_csr_build", "fr_solver_create", "fr_solver_run", "fr_power_run", "fr_pagerank_host"} <= names


def test_library_exports_every_declared_symbol():
    from paper_1202_6158_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers exactly the declared set
    assert set(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_no_device_here():
    import torch
    from paper_1202_6158_b200 import _lib
    assert _lib.lib.fr_abi_version() == 3
    if not torch.cuda.is_available():
        assert _lib.lib.fr_device_sms() == 0
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _lib.require_device()


def test_library_is_sm100a():
    """The shipped kernels are sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_1202_6158_b200 import _lib
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    """The oracle is test infrastructure: no product source imports it, loads its
    library (a ctypes load of oracle/libfr_oracle.so would bypass an import check)
    or names its directory."""
    pkg = os.path.join(ROOT, "paper_1202_6158_b200")
    sources = glob.glob(os.path.join(pkg, "*.py")) + glob.glob(os.path.join(pkg, "csrc", "*.cu")) + \
        glob.glob(os.path.join(pkg, "csrc", "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    assert len(sources) >= 15
    for path in sources:
        src = open(path).read()
        assert "import oracle" not in src and "from oracle" not in src, path
        # code only: comments and docstrings may cite the oracle's generator spec
        if path.endswith(".py"):
            code = re.sub(r'(""".*?"""|#[^\n]*)', "", src, flags=re.S)
        else:
            code = re.sub(r"(/\*.*?\*/|//[^\n]*)", "", src, flags=re.S)
        assert "oracle" not in code, path


def _c_layout(struct, fields, tmp_path):
    """sizeof / offsetof of a header struct, from a tiny C program compiled with gcc."""
    import subprocess
    src = tmp_path / "layout.c"
    body = "".join(f'printf("%zu ", offsetof({struct}, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "fluidrank_b200.h"\n'
                   f'int main(void) {{ printf("%zu ", sizeof({struct})); {body} return 0; }}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    return [int(x) for x in out]


@pytest.mark.parametrize("name,struct", [("SolverConfig", "fr_solver_config"), ("SolveStats", "fr_solve_stats"),
                                         ("TraceRow", "fr_trace_row"), ("GenConfig", "fr_gen_config")])
def test_ctypes_structs_match_the_header(tmp_path, name, struct):
    """The ctypes mirrors in _lib.py have the C layout (sizes and every field offset)."""
    from paper_1202_6158_b200 import _lib
    cls = getattr(_lib, name)
    fields = [f[0] for f in cls._fields_]
    c = _c_layout(struct, fields, tmp_path)
    py = [ctypes.sizeof(cls)] + [getattr(cls, f).offset for f in fields]
    assert c == py


def test_integration_stub_matches_the_library():
    """The ctypes stub shown in INTEGRATION.md declares the same struct layouts."""
    from paper_1202_6158_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    ns = {"ctypes": ctypes}
    exec(text[text.index("class SolverConfig"):text.index("_lib.fr_pagerank_host.argtypes")], ns)
    for name in ("SolverConfig", "SolveStats"):
        assert ns[name]._fields_ == getattr(_lib, name)._fields_, name
