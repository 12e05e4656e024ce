"""Module-level drop-in: make `import cutbench` (and its submodules) resolve to
this package, so code written against the reference runs unchanged.

    import paper_2603_01443_b200 as b200
    b200.install_as_cutbench()
    from cutbench.harness import measure, sweep_heatmap    # GPU-backed
    from cutbench.costmodel import threshold_uniform

Mapping (reference module -> this package, `/root/reference/pkg/src/cutbench/`):
circuits, cutting, engine, merging, errors, cli -> same names; costmodel ->
theory; svmfit -> boundary_fit; harness -> harness + sweeps (one namespace).
"""
from __future__ import annotations

import sys
import types


def install_as_cutbench(name: str = "cutbench", *, replace: bool = False) -> types.ModuleType:
    """Register this package under `name` in sys.modules (refuses to shadow an
    already-imported module of that name unless replace=True)."""
    import paper_2603_01443_b200 as pkg

    from . import boundary_fit, circuits, cli, cutting, engine, errors, harness, merging, sweeps, theory

    cur = sys.modules.get(name)
    if cur is not None and getattr(cur, "__dropin_of__", None) is not pkg and not replace:
        raise RuntimeError(f"module {name!r} is already imported; pass replace=True to shadow it")
    combined = types.ModuleType(f"{name}.harness", harness.__doc__)
    for mod in (harness, sweeps):
        for attr, val in vars(mod).items():
            if not attr.startswith("__"):
                setattr(combined, attr, val)
    subs = {"circuits": circuits, "cutting": cutting, "engine": engine, "merging": merging, "errors": errors,
            "cli": cli, "costmodel": theory, "svmfit": boundary_fit, "harness": combined}
    # a proxy package: the package's public names, with the submodule
    # attributes pointing at the reference-named modules (so both
    # `import cutbench.harness` and `from cutbench import harness` see the
    # combined harness namespace)
    proxy = types.ModuleType(name, pkg.__doc__)
    for attr, val in vars(pkg).items():
        if not attr.startswith("__"):
            setattr(proxy, attr, val)
    for sub, mod in subs.items():
        setattr(proxy, sub, mod)
    proxy.__path__ = []  # a package: submodules resolve through sys.modules
    proxy.__dropin_of__ = pkg
    sys.modules[name] = proxy
    for sub, mod in subs.items():
        sys.modules[f"{name}.{sub}"] = mod
    return proxy
