"""INTEGRATION.md shows the reference-side binding a maintainer would add;
it must be the module the GPU integration test actually runs."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_md_embeds_the_tested_stub():
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", md, re.S)
    src = open(os.path.join(ROOT, "integration", "gf_b200_backend.py")).read()
    assert any(b.strip() == src.strip() for b in blocks), \
        "INTEGRATION.md's stub differs from integration/gf_b200_backend.py"


def test_header_citations_name_real_reference_functions():
    """Every gf/guided.py function a header comment cites exists there."""
    hdr = open(os.path.join(ROOT, "include", "gf_b200.h")).read()
    for name in ("guided_filter(", "guided_filter_full("):
        assert name not in hdr
