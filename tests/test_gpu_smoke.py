"""The driver's round-end smoke (__graft_entry__.smoke) runs as a GPU test too,
so a regression in it (e.g. a broadcasting shape bug that exhausts host
memory) shows up in `pytest -m gpu` first."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_smoke():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import __graft_entry__
    __graft_entry__.smoke()
