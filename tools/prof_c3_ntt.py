"""One C3 run_report (staged: 256 entry grids of 64^3 per prime) and one C5
prime step, for an ncu launch list with DRAM bytes per kernel:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/ntt_launches.csv python tools/prof_c3_ntt.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2010_12117_b200 import executor, plan, run_report, workloads  # noqa: E402

m, cfg = workloads.c3()
run_report(m, cfg)
m5, cfg5 = workloads.c5()
pl5 = plan(m5, cfg5)
st = executor.PrimeStages(m5, pl5, staged=False)
st.forward(0)
st.det_kernels(0)
st.expand(0)
st.interpolate(0)
torch.cuda.synchronize()
