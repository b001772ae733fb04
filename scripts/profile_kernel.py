"""Launch one kernel config a few times for ncu (run under `ncu ... python scripts/profile_kernel.py`).

    ncu --set full --clock-control none --import-source on -k regex:conv2d -s 2 -c 1 \
        -o gpurun_out/conv2d python scripts/profile_kernel.py conv2d
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main():
    name = sys.argv[1]
    objective = sys.argv[2] if len(sys.argv) > 2 else "time_optimal"
    overrides = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
    gpu = GPU(0)
    p = make_problem(name)
    p.prepare(gpu)
    cfg = {**(tuned.best_config(name, objective) or p.default_config()), **overrides}
    k = p.kernel(cfg)
    p.bind(k, cfg)
    for _ in range(5):
        gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    print(json.dumps({"kernel": name, "config": cfg, "regs": k.regs, "smem": k.static_smem}))
    gpu.close()


if __name__ == "__main__":
    main()
