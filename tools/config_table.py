"""Per-config bench table (markdown) from the JSON lines of tools/gpu_artifacts.sh.

usage: python tools/config_table.py gpurun_out/<TAG> > table.md
Reads bench_cfg2.json (headline) and bench_<config>.json for every config."""
import json
import os
import sys

ORDER = ["cfg2", "cfg1", "cfg3-zf", "cfg3-mrc", "cfg4-fd", "cfg4-pd", "cfg5-pd512", "cfg5-fd512", "cfg5-pd1024",
         "cfg5-fd1024"]


def last_json(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    d = sys.argv[1]
    print("| workload | Gb/s | ms/step | frac of HBM | kernel(s) | x-hat err | sigma2 err | decision mismatches | clocks |")
    print("|---|---|---|---|---|---|---|---|---|")
    for c in ORDER:
        p = os.path.join(d, f"bench_{c}.json")
        if not os.path.exists(p):
            continue
        j = last_json(p)
        if j is None:
            continue
        par = j.get("parity") or {}
        clk = j.get("clocks") or {}
        print(f"| {j['config']['workload']} | {j['value']:.2f} | {j['ms_per_step']:.4f} | "
              f"{j['roofline']['frac']:.3f} | {j['roofline']['kernel']} | "
              f"{par.get('xhat_normwise_max', float('nan')):.1e} | {par.get('sigma2_entry_max', float('nan')):.1e} | "
              f"{par.get('decision_mismatches', '-')} / {par.get('symbols_checked', '-')} | "
              f"{clk.get('sm_mhz', '-')} MHz {','.join(clk.get('reasons', []))} |")


if __name__ == "__main__":
    main()
