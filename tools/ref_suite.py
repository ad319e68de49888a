"""Run the REFERENCE's own hot-path test files, unmodified, against the drop-in.

    # build container: stage a copy of the reference tests (git-ignored; it
    # travels to the GPU box with the gpurun snapshot like baseline/_ref)
    python tools/ref_suite.py --stage
    # GPU box: run them with ``import ldurepart`` aliased to this package
    python tools/ref_suite.py [pytest args] [--files test_repart.py ...]

The alias maps ``ldurepart`` and its submodules (core, repart, update, solver,
transport, assembly) to paper_2510_08536_b200; the reference's own cli.py and
costmodel.py (out of scope) are loaded unmodified as submodules of the alias,
so test_acceptance's case sweeps drive the B200 path.  The reference's verification helpers
(``ldurepart.oracle``: reference_global_assemble, compare_matrices, to_csr,
...) are checkers, out of this repo's scope; they are taken
from the unmodified reference installed in baseline/_ref.  Nothing in the
product path imports this file.
"""

import argparse
import importlib.util
import os
import shutil
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = os.path.join(ROOT, "baseline", "_ref_tests")
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "ldurepart")
# hot-path files (the parity contract) plus the formats, generator,
# transport and acceptance files whose subjects the drop-in re-implements;
# test_oracle / test_costmodel / test_cli cover out-of-scope modules
FILES = ["test_core.py", "test_assembly.py", "test_transport.py", "test_repart.py",
         "test_update.py", "test_solver.py", "test_acceptance.py"]


def stage():
    src = "/root/reference/pkg/tests"
    if os.path.exists(STAGE):
        shutil.rmtree(STAGE)
    shutil.copytree(src, STAGE, ignore=shutil.ignore_patterns("__pycache__"))
    print(f"staged {src} -> {STAGE}")


def _load_reference_package():
    """The unmodified reference as package ``_ldurepart_ref`` (for its oracle)."""
    spec = importlib.util.spec_from_file_location(
        "_ldurepart_ref", os.path.join(REF_PKG, "__init__.py"),
        submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_ldurepart_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def install_alias():
    sys.path.insert(0, ROOT)
    import paper_2510_08536_b200 as lrb
    import importlib
    # submodules by import path (the package namespace re-exports functions of
    # the same names, e.g. update)
    core, repart, solver, transport, update = (
        importlib.import_module(f"paper_2510_08536_b200.{m}")
        for m in ("core", "repart", "solver", "transport", "update"))
    ref = _load_reference_package()
    alias = types.ModuleType("ldurepart")
    alias.__dict__.update({k: v for k, v in vars(lrb).items() if not k.startswith("__")})
    alias.__path__ = []
    oracle = sys.modules["_ldurepart_ref.oracle"]
    for name in ("reference_global_assemble", "assemble_global_from_parts", "compare_matrices",
                 "reference_solve", "to_csr"):
        if not hasattr(alias, name):
            setattr(alias, name, getattr(oracle, name))
    alias.oracle = oracle
    sys.modules["ldurepart"] = alias
    cavity = importlib.import_module("paper_2510_08536_b200.cavity")
    for name, mod in (("core", core), ("repart", repart), ("solver", solver),
                      ("transport", transport), ("update", update), ("oracle", oracle),
                      ("assembly", cavity)):
        sys.modules[f"ldurepart.{name}"] = mod
        if not hasattr(alias, name):   # lr.update stays the function, as in the reference
            setattr(alias, name, mod)
    # the reference's driver and cost model (out of this repo's scope, SURVEY
    # §2) are loaded from its unmodified sources AS submodules of the alias,
    # so their relative imports (.repart, .update, .solver, ...) bind to the
    # drop-in: test_acceptance's sweeps run the B200 path end to end
    for name in ("costmodel", "cli"):
        spec = importlib.util.spec_from_file_location(f"ldurepart.{name}",
                                                      os.path.join(REF_PKG, f"{name}.py"))
        mod = importlib.util.module_from_spec(spec)
        mod.__package__ = "ldurepart"
        sys.modules[f"ldurepart.{name}"] = mod
        spec.loader.exec_module(mod)
        setattr(alias, name, mod)
    # the names the reference's __init__ re-exports from them (__init__.py:25-33)
    for name in ("CappedSpeedup", "CommCostParams", "CostCurves", "DegradingSpeedup",
                 "IdealSpeedup", "Resources", "TabulatedSpeedup", "best_homogeneous",
                 "load_curves_csv", "optimize_ranks", "recommend_alpha", "total_time",
                 "total_time_hetero"):
        if not hasattr(alias, name):
            setattr(alias, name, getattr(sys.modules["ldurepart.costmodel"], name))
    for name in ("BenchRecord", "CaseConfig", "run_case", "sweep"):
        if not hasattr(alias, name):
            setattr(alias, name, getattr(sys.modules["ldurepart.cli"], name))
    return ref


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("--files", nargs="*", default=FILES)
    args, rest = ap.parse_known_args()
    if args.stage:
        stage()
        return 0
    if not os.path.isdir(STAGE):
        raise SystemExit("reference tests not staged: run tools/ref_suite.py --stage in the build "
                         "container first")
    install_alias()
    sys.path.insert(0, STAGE)
    import pytest
    return pytest.main(["-p", "no:cacheprovider", "--rootdir", STAGE, "-c", os.devnull,
                        *[os.path.join(STAGE, f) for f in args.files], *rest])


if __name__ == "__main__":
    sys.exit(main())
