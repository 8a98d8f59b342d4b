"""pytest plugin: run the reference's OWN test files, unchanged, against the
drop-in (`-p _refsuite`, used by tests/test_reference_suite.py).

The reference tests import `packtrain.{packing,engine,data,tuner,device_sim}`.
This plugin makes `packtrain` resolve to `paper_2002_02885_b200` before they
are collected:

- `packtrain.packing`, `.data`, `.engine` are the drop-in modules themselves;
- `packtrain.tuner` is the drop-in `tuner` module, plus the names that the
  reference defines on top of its P5000 simulator (`SimulatedExecutor`,
  `model_profile_for`, `make_traintime_metric`; reference tuner.py:118-139,
  :369-417), which are out of scope here and are taken from the
  installed, unmodified reference in `baseline/_ref`. The reference's
  `EngineExecutor` (tuner.py:420-483) maps to `tuner.B200Executor`, its drop-in;
- `packtrain.device_sim` is the reference's own simulator module from
  `baseline/_ref` (out of scope: the tests use it only as a cost oracle / byte
  accountant), with its `OOMError` bound to the drop-in's
  `device.OOMError` (same constructor, device_sim.py:23-30) so the simulator
  and the drop-in's packer raise, and the tests catch, one class.

The reference package is loaded under the private name `_packtrain_ref` so the
two never shadow each other. Its simulator reads `.profile` files with
`importlib.resources.files("packtrain")`; that lookup is pointed at the
reference's own directory (in memory, nothing on disk changes).

Test infrastructure only: nothing in `paper_2002_02885_b200/` imports this.
"""
import importlib.util
import os
import pathlib
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "packtrain")


def _load_reference():
    if "_packtrain_ref" in sys.modules:
        return sys.modules["_packtrain_ref"]
    spec = importlib.util.spec_from_file_location(
        "_packtrain_ref", os.path.join(REF_PKG, "__init__.py"),
        submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_packtrain_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def _ref_submodule(name):
    _load_reference()
    return importlib.import_module(f"_packtrain_ref.{name}")


def install():
    if sys.modules.get("packtrain") is not None and \
            getattr(sys.modules["packtrain"], "__refsuite__", False):
        return
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_2002_02885_b200 as dropin
    from paper_2002_02885_b200 import data, device, engine, packing, tuner

    dev = _ref_submodule("device_sim")
    ref_dir = pathlib.Path(REF_PKG)
    dev.resources = types.SimpleNamespace(files=lambda _pkg: ref_dir)
    dev.OOMError = device.OOMError  # one OOM class on both sides (same signature)
    mods = {"packing": packing, "device_sim": dev}
    for name, ours in (("engine", engine), ("data", data), ("tuner", tuner)):
        ref = _ref_submodule(name)
        shim = types.ModuleType(f"packtrain.{name}")
        shim.__dict__.update({k: v for k, v in vars(ours).items() if not k.startswith("__")})
        shim.__doc__ = ours.__doc__
        for k, v in vars(ref).items():
            if not k.startswith("_") and not hasattr(ours, k) and not isinstance(v, types.ModuleType):
                setattr(shim, k, v)
                INJECTED.append(f"{name}.{k}")
        mods[name] = shim
    mods["tuner"].EngineExecutor = tuner.B200Executor

    pkg = types.ModuleType("packtrain")
    pkg.__path__ = []
    pkg.__refsuite__ = True
    pkg.__version__ = dropin.__version__
    for name, mod in mods.items():
        setattr(pkg, name, mod)
        sys.modules[f"packtrain.{name}"] = mod
    sys.modules["packtrain"] = pkg


# Reference tests that would exercise only reference code injected above (its
# host numpy engine, file loaders, CLI and simulator) or the P5000 memory model:
DESELECT = {
    "test_pack.py::test_load_model_registers_memory_on_device":
        "asserts the P5000 simulator's byte model (a 6-8-3 MLP > 150 MB); the drop-in "
        "registers the member's real B200 slab bytes (device.member_device_bytes)",
    "test_acceptance.py::test_criterion_01_gradient_oracle":
        "the host numpy engine (forward/backward): the oracle's role here (oracle/mlp64.py)",
    "test_acceptance.py::test_criterion_05_metrics_algebra": "CLI + simulator (out of scope)",
    "test_acceptance.py::test_criterion_08_simulator_qualitative": "simulator only (out of scope)",
    "test_data.py::test_binary_round_trip": "PTDS loader (out of scope)",
    "test_data.py::test_csv_loading": "CSV loader (out of scope)",
    "test_data.py::test_malformed_files_are_rejected": "PTDS/CSV loaders (out of scope)",
}
INJECTED: list = []


def pytest_configure(config):
    install()


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        key = f"{it.path.name}::{getattr(it, 'originalname', it.name)}"
        (drop if key in DESELECT else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep


def pytest_report_header(config):
    return [f"refsuite: packtrain -> paper_2002_02885_b200; reference names injected "
            f"(out of scope): {', '.join(INJECTED)}"]
