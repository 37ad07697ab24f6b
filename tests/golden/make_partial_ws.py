"""Write a reference-produced, partially completed workspace as a fixture
(run here, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_partial_ws.py

The reference run is killed after its 7th progress unit; the directory
`tests/golden/ref_partial_ws/` (+ `ref_partial_ws.json` with the expected
result and the units still to do) lets the GPU tests resume it with this
package (cross-resume)."""
import json
import random
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
import polydet as ref  # noqa: E402
from oracles import random_matrix_terms  # noqa: E402


class Stop(Exception):
    pass


def main():
    rows = random_matrix_terms(random.Random(21), 3, 2, 2, 30, 3)
    m = ref.poly_matrix(rows, ("x", "y"))
    full_units = []
    result = ref.run(m, ref.PipelineConfig(progress=full_units.append))
    out = HERE / "ref_partial_ws"
    shutil.rmtree(out, ignore_errors=True)
    seen = []

    def cb(unit):
        seen.append(unit)
        if len(seen) == 7:
            raise Stop()

    try:
        ref.run(m, ref.PipelineConfig(progress=cb), workspace=out)
    except Stop:
        pass
    (HERE / "ref_partial_ws.json").write_text(json.dumps({
        "input": m.to_dict(), "done_units": seen, "remaining_units": full_units[len(seen):],
        "terms": [[list(e), int(c)] for e, c in sorted(result.terms().items())], "shape": list(result.shape)}))
    print("wrote", out, sorted(p.name for p in out.iterdir()))


if __name__ == "__main__":
    main()
