"""pytest plugin (``-p reference_overlay_plugin``, this directory on PYTHONPATH), loaded only by tests/test_gpu_reference_suite.py in a child
pytest that runs the REFERENCE's own test-suite: before the reference's test modules are imported, every function
of ``tetipc`` that ``paper_2308_09400_b200`` mirrors is swapped for the mirror
(``paper_2308_09400_b200.integration.function_overlay``).  Writes the per-function call counts to
``$B200_OVERLAY_REPORT`` when the session ends.  ``$B200_OVERLAY_BATCHED``: the reference's ``SimState`` is the batched
subclass of ``integration.b200_sim_state`` as well."""

import json
import os

_STATE = {}


def pytest_configure(config):
    import tetipc
    import tetipc.barrier, tetipc.elasticity, tetipc.friction, tetipc.gap, tetipc.kernels  # noqa: F401,E401
    import tetipc.mollifier, tetipc.proximity, tetipc.solver  # noqa: F401,E401

    from paper_2308_09400_b200 import integration

    _STATE["calls"] = {}
    _STATE["cm"] = integration.function_overlay(tetipc, _STATE["calls"], batched=bool(os.environ.get("B200_OVERLAY_BATCHED")))
    _STATE["cm"].__enter__()


def pytest_unconfigure(config):
    cm = _STATE.pop("cm", None)
    if cm is not None:
        cm.__exit__(None, None, None)
    path = os.environ.get("B200_OVERLAY_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump(_STATE.get("calls", {}), fh, indent=1, sort_keys=True)
