"""pytest plugin: run the REFERENCE's own test modules with the B200 backend
installed at its joint-layer seam (integration/gf_b200_backend.py, the stub
INTEGRATION.md documents).  Loaded with ``-p ref_b200_plugin`` by
tests/test_gpu_integration.py; writes the backend's call counts to
$GF_B200_CALLS at the end so the caller can see the kernels really ran."""

import json
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_ROOT, "baseline", "_ref"))
sys.path.insert(0, _ROOT)

import guidedfilter  # noqa: E402
import guidedfilter.verify  # noqa: E402,F401  (loaded so its imports get patched too)
import guidedfilter.training  # noqa: E402,F401

from integration import gf_b200_backend as backend  # noqa: E402

backend.install(guidedfilter)


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("GF_B200_CALLS")
    if path:
        with open(path, "w") as f:
            json.dump(backend.CALLS, f)
