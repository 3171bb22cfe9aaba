"""libtlgpu.so builds for sm_100a, loads, and exports every symbol include/tlgpu.h declares.

CPU-only: no compute call is made (there is no GPU in the build container).
"""

import ctypes
import re
import subprocess

import numpy as np
import pytest

from paper_2110_12932_b200 import _native as N
from paper_2110_12932_b200.build import OUT, build

from .conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "tlgpu.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(tl_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    return build()


def test_library_exports_header_symbols(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    declared = header_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes binding covers exactly the header
    assert sorted(n for n, _, _ in N.SIGNATURES) == declared


def test_binding_loads_and_reports_abi(lib_path):
    lib = N.lib()
    assert lib.tl_abi_version() == N.ABI_VERSION


def test_plan_struct_layouts_match_header():
    assert N.MACRO_DTYPE.itemsize == ctypes.sizeof(N.MacroPlan) == 64
    assert N.MICRO_DTYPE.itemsize == ctypes.sizeof(N.MicroPlan) == 48


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setenv("TLGPU_LIB", str(tmp_path / "missing.so"))
    with pytest.raises(N.NativeLibraryMissing):
        N.lib()
    monkeypatch.setattr(N, "_lib", None)


def test_struct_layouts_match_c_compiler(tmp_path):
    """sizeof / offsetof of every ABI struct as gcc lays them out == the ctypes mirror."""
    structs = {"tl_solve_info": N.SolveInfo, "tl_grid_desc": N.GridDesc, "tl_gaussian": N.Gaussian,
               "tl_run_desc": N.RunDesc, "tl_macro_plan": N.MacroPlan, "tl_micro_plan": N.MicroPlan,
               "tl_slab": N.Slab}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT / "include" / "tlgpu.h"}"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname} {fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_cli_parser_and_config_error(tmp_path, capsys):
    """lpbfsim/cli.py's interface: run / study / compare subcommands; a bad config exits 2."""
    from paper_2110_12932_b200.cli import build_parser, main
    p = build_parser()
    a = p.parse_args(["compare", "configs/cfg1_compare.cfg", "--out", str(tmp_path), "--snapshots", "none"])
    assert a.command == "compare" and a.snapshots == "none" and a.out == tmp_path
    assert main(["run", str(tmp_path / "missing.cfg")]) == 2
    assert "config error" in capsys.readouterr().err


def test_vtk_writer_matches_reference_file(tmp_path):
    """experiment.write_vtk (vtkio.write_vtk, vtkio.py:15-44): the reference's own file for a
    translated 5 x 3 x 3-cell mesh, byte for byte (element order, orientation flips, format)."""
    import numpy as np
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.experiment import write_vtk
    from .conftest import GOLDEN
    g = P.build_structured_grid(P.Box((1e-4, 2e-4, 0.0), (3.5e-4, 3.5e-4, 1.5e-4)), 5e-5).translated(
        (1e-5, -2e-5, 0.0))
    write_vtk(tmp_path / "s.vtk", g, {"temperature": np.load(GOLDEN / "small_vtk_field.npy")})
    assert (tmp_path / "s.vtk").read_text() == (GOLDEN / "small.vtk").read_text()
