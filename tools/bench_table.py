"""Print the per-layer breakdown of a bench.py JSON line.
usage: python tools/bench_table.py bench_output.log"""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print({k: d[k] for k in ("value", "unit", "n_gpus", "ms_per_step", "gpu_launches") if k in d})
    print("roofline", d.get("roofline"))
    print("e2e", d.get("e2e"), "clocks", d.get("clocks"))
    tot = {"fwd": 0, "bn": 0, "bpw": 0, "bpx": 0}
    for l in d["config"].get("layers", []):
        if not isinstance(l, dict):
            continue
        print(f'{l["name"]:8s} {str(l["shape_NCHW_F_K_S_P"]):38s} {str(l["decomp"]):10s} fwd {l["fwd_ms"]*1e3:7.1f}'
              f' bn {l["bn_stats_ms"]*1e3:6.1f} bpw {l["bwd_filter_ms"]*1e3:7.1f} bpx {l["bwd_data_ms"]*1e3:7.1f} us'
              f'  fwdTF {l["fwd_tflops"]:6.0f} bwdTF {l["bwd_tflops"]:6.0f}')
        tot["fwd"] += l["fwd_ms"]; tot["bn"] += l["bn_stats_ms"]; tot["bpw"] += l["bwd_filter_ms"]; tot["bpx"] += l["bwd_data_ms"]
    print("totals ms", {k: round(v, 3) for k, v in tot.items()})
