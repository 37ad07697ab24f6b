"""Cross-resume fixtures, CPU side.

tests/golden/ref_partial_ws/   written by the reference, killed after 7 units
                               (tests/golden/make_partial_ws.py)
tests/golden/b200_partial_ws/  written by this package on a B200, killed after
                               the same 7 units (tools/write_partial_ws.py)

The two directories are byte-identical; the reference finishes the one this
package wrote (when /root/reference is present, i.e. in the build container),
and tests/test_gpu_parity.py::test_resume_reference_written_partial_workspace
covers the other direction on the GPU."""

import hashlib
import json
import shutil
import sys
from pathlib import Path

import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def _hashes(d):
    return {q.name: hashlib.sha256(q.read_bytes()).hexdigest() for q in sorted(d.iterdir())}


def test_partial_workspaces_byte_identical():
    ours, theirs = _hashes(GOLDEN / "b200_partial_ws"), _hashes(GOLDEN / "ref_partial_ws")
    assert len(ours) == 10
    assert ours == theirs


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference sources not present")
def test_reference_resumes_b200_written_workspace(tmp_path):
    sys.path.insert(0, str(REFERENCE_SRC))
    try:
        import polydet as ref
    finally:
        sys.path.remove(str(REFERENCE_SRC))
    meta = json.loads((GOLDEN / "ref_partial_ws.json").read_text())
    ws = tmp_path / "ws"
    shutil.copytree(GOLDEN / "b200_partial_ws", ws)
    seen = []
    got = ref.resume(ws, ref.PipelineConfig(progress=seen.append))
    assert seen == meta["remaining_units"]
    assert got.terms() == {tuple(e): c for e, c in meta["terms"]}
