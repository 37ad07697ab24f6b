"""Write a workspace with THIS package (GPU) and kill the run after its 7th
unit, for the reverse cross-resume fixture (the reference finishes it in
tests/test_cross_resume.py):

    python tools/write_partial_ws.py gpurun_out/b200_partial_ws
"""
import json
import random
import shutil
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2010_12117_b200 import PipelineConfig, PolyMatrix, run  # noqa: E402


class Stop(Exception):
    pass


def main(out):
    meta = json.loads((Path(__file__).resolve().parents[1] / "tests/golden/ref_partial_ws.json").read_text())
    m = PolyMatrix.from_dict(meta["input"])
    out = Path(out)
    shutil.rmtree(out, ignore_errors=True)
    seen = []

    def cb(unit):
        seen.append(unit)
        if len(seen) == 7:
            raise Stop()

    try:
        run(m, PipelineConfig(progress=cb), workspace=out)
    except Stop:
        pass
    print("done units", seen, sorted(p.name for p in out.iterdir()))


if __name__ == "__main__":
    main(sys.argv[1])
