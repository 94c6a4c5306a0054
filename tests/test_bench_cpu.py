"""bench.py's reference arm (CPU fp32 oracle on the host cores) prints the contract's JSON line:
same metric / unit / direction as the GPU arm, impl "reference", a cpu_baseline describing the
sample and an e2e with no host<->device bytes; plus the directly timed C1 iteration."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    import bench  # noqa: E402  (the arm's metric string)

    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "tokens/s" and line["higher_is_better"] is True and line["scaling"] == "strong"
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    c1 = line["c1_iteration"]
    assert c1["config"] == "C1" and c1["ms"] > 0 and c1["loss"] > 0
    assert line["config"]["workload"] == "C2"
