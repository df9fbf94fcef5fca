"""Test infrastructure: route the vendored reference's hot-path names to the
drop-in package (`python -m pytest -p ref_swap ...` or `ref_swap.install()`).

Every public name of roboserve.{core, horizon, waiting, engines, scheduler,
workload} that the drop-in also defines (functions and value types) is
replaced in the reference module's namespace -- and in the reference modules
that imported it by name (sim.py binds `plan` at import) -- so the reference's
own tests and scripts, which import those names from `roboserve.*`, exercise
the CUDA path.  Names the drop-in does not implement (the simulator, the CLI,
poisson_arrivals) stay the reference's.  baseline/_ref is vendored by
tools/vendor_reference.sh; nothing here is imported by the product."""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
MODULES = ("core", "horizon", "waiting", "engines", "scheduler", "workload")


def available() -> bool:
    return (REF / "roboserve" / "__init__.py").exists()


def install() -> list[str]:
    """Patch the reference modules; returns the swapped qualified names."""
    for p in (str(REF), str(ROOT)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import paper_2605_11381_b200 as kb
    swapped = []
    mods = {m: importlib.import_module(f"roboserve.{m}") for m in MODULES}
    extra = [importlib.import_module(f"roboserve.{m}") for m in ("sim", "experiments", "cli")]
    for name, mod in mods.items():
        for attr in list(vars(mod)):
            if attr.startswith("_") or not hasattr(kb, attr):
                continue
            ref_obj = getattr(mod, attr)
            if getattr(ref_obj, "__module__", "").split(".")[0] != "roboserve":
                continue  # re-exported third-party names (np, dataclass, ...)
            ours = getattr(kb, attr)
            setattr(mod, attr, ours)
            swapped.append(f"{name}.{attr}")
            for m2 in list(mods.values()) + extra + [importlib.import_module("roboserve")]:
                if getattr(m2, attr, None) is ref_obj:
                    setattr(m2, attr, ours)
    return swapped


def pytest_configure(config):  # -p ref_swap
    install()
