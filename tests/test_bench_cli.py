"""bench.py contract on CPU: the reference arm (the fp64 oracle, PAPER.md
Eq. 1 / 2 / 3 timed on host cores) prints exactly ONE JSON line on stdout
with the keys the driver reads; everything else goes to stderr."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-budget", "0.3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3
    assert d["unit"] == "TFLOP/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "mesh2k_n8"


def test_resnet50_conv_stack_workload():
    """The ResNet-50 conv-stack proxy (BASELINE.json configs[2]): 53
    convolutions with Caffe's stride placement, 7.71 GFLOP per 224^2 image
    forward (reading R21)."""
    import bench
    L = bench.resnet50_convs(1)
    assert len(L) == 53
    assert abs(sum(bench.layer_flops(l) for l in L) / 1e9 - 7.7118) < 1e-3
    # the last stage runs at 7x7, the 3x3s have stride 1 and pad 1
    assert all(l[3] == 7 for l in L if l[0].startswith("res5") and "branch2a" not in l[0] and "branch1" not in l[0])
    assert all(l[6] == 3 and l[7] == 1 and l[8] == 1 for l in L if l[0].endswith("branch2b"))
    assert bench.WORKLOADS["resnet50_n64"][0][1] == 64
