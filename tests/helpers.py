"""Shared test helpers: repo paths and golden-fixture loading."""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def golden(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip("golden fixture %s not generated" % name)
    return json.loads(path.read_text())
