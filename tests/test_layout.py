"""Repository rules that keep the product honest: the package never imports
the oracle (test infrastructure), has no Triton/torch.compile path, and the
reference's module names exist for the drop-in alias."""
import os
import re
import sys

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2603_01443_b200")


def _sources():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".h")):
                yield os.path.join(dirpath, f)


def test_product_never_imports_the_oracle():
    pat = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b)|cutbench_oracle|oracle_c\b", re.M)
    for path in _sources():
        assert not pat.search(open(path).read()), path


def test_no_compat_layers():
    pat = re.compile(r"import\s+triton|torch\.compile|tilelang")
    for path in _sources():
        assert not pat.search(open(path).read()), path


def test_module_alias_switch():
    import paper_2603_01443_b200 as b200

    saved = {k: v for k, v in sys.modules.items() if k == "cutbench" or k.startswith("cutbench.")}
    try:
        for name in ("circuits", "engine", "cutting", "merging", "errors"):
            sys.modules[f"cutbench.{name}"] = getattr(b200, name)
        sys.modules["cutbench"] = b200
        from cutbench.circuits import BenchmarkSpec, build_staircase  # noqa: PLC0415
        from cutbench.cutting import decompose, plan_cut  # noqa: PLC0415
        from cutbench.merging import MergeInput, merge, merge_input_from  # noqa: F401,PLC0415

        circ = build_staircase(BenchmarkSpec(q=6, n=3, blocks=2))
        subs = decompose(circ, plan_cut(circ, 3))
        assert subs.num_subcircuits == 4 + 16 + 4
    finally:
        for k in [k for k in sys.modules if k == "cutbench" or k.startswith("cutbench.")]:
            del sys.modules[k]
        sys.modules.update(saved)
