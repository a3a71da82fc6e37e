"""Monte Carlo SER driver on the GPU vs the reference path on the host cores,
on acceptance criterion 8's experiment set (reference test_acceptance.py:
174-207): B=256, U=16, C=8, 16-QAM, SNR 9.5 / 11 / 12.5 dB, 2000 trials,
MRC / ZF / L-MMSE / LAMA x PD / FD, seed 1.

GPU: paper_1808_04473_b200.montecarlo.run_experiment (host NumPy draws,
bit-identical to the reference's, shared by the 8 experiments; one fused
launch per SNR point; plus the analytic ser_predicted); the throughput
figure times the detection alone (count_errors), like the CPU side.  CPU: the reference's per-trial path (the oracle
port, oracle/dbp_oracle.py) on a bounded sample of trials over all host
cores, extrapolated to the full set.  Prints one JSON line.

usage: python tools/mc_bench.py [--trials 2000] [--cpu-trials 24]
"""

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

KINDS = ("mrc", "zf", "lmmse", "lama")
ARCHS = ("pd", "fd")
SNR = (9.5, 11.0, 12.5)


def _cpu_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, REPO)
    from oracle import dbp_oracle as O

    kind, arch, H, Y, n0, offs, syms = args
    fn = O.fd_equalize if arch == "fd" else O.pd_equalize
    lp = {"t_max": 10} if kind == "lama" else None
    for n in range(H.shape[0]):
        r = fn(kind, H[n].astype(complex), Y[n, 0].astype(complex), offs, n0, 1.0, syms, lp)
        O.hard_detect_index(r["z"], syms)
    return H.shape[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=2000)
    ap.add_argument("--cpu-trials", type=int, default=1600)
    args = ap.parse_args()
    import torch

    import paper_1808_04473_b200 as dbp
    from paper_1808_04473_b200 import montecarlo as mc

    q16 = dbp.make_constellation("qam16")
    part = dbp.ClusterPartition.uniform(256, 8)

    def cfg(kind, arch):
        return mc.ExperimentConfig(b=256, u=16, constellation=q16, partition=part, equalizer=kind,
                                   architecture=arch, snr_db=SNR, trials=args.trials, seed=1, lama_t_max=10)

    t0 = time.perf_counter()
    inputs = [mc.draw_inputs(cfg("zf", "pd"), k) for k in range(len(SNR))]
    t_draw = time.perf_counter() - t0
    mc.run_experiment(cfg("lmmse", "pd"), inputs=inputs)  # warm-up (library load, first launches)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    results = {(k, a): mc.run_experiment(cfg(k, a), inputs=inputs) for k in KINDS for a in ARCHS}
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t0  # incl. the analytic predictions (LAMA fixed points)
    t0 = time.perf_counter()  # detection only: the part the CPU baseline times
    for k in KINDS:
        for a in ARCHS:
            for inp in inputs:
                mc.count_errors(cfg(k, a), inp)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    n_exp_trials = len(KINDS) * len(ARCHS) * len(SNR) * args.trials
    # orderings of criterion 8 (test_acceptance.py:189-207), CI overlap
    ok = True
    for arch in ARCHS:
        for i in range(len(SNR)):
            r = {k: results[k, arch].points[i] for k in KINDS}
            ok &= r["lama"].ci_low <= r["lmmse"].ci_high and r["lmmse"].ci_low <= r["zf"].ci_high
            if arch == "pd":
                ok &= r["zf"].ci_high < r["mrc"].ci_low
    for k in KINDS:
        for i in range(len(SNR)):
            ok &= results[k, "pd"].points[i].ci_low <= results[k, "fd"].points[i].ci_high
    # CPU: reference path per trial on a bounded sample, all host cores
    cores = os.cpu_count() or 1
    offs = list(part.offsets)
    jobs = []
    per = max(1, args.cpu_trials // cores)
    for k in KINDS:
        for a in ARCHS:
            inp = inputs[1]
            for c in range(cores):
                sl = slice(c * per, (c + 1) * per)
                jobs.append((k, a, inp.h[sl], inp.y[sl], inp.n0, offs, q16.symbols))
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_cpu_worker, jobs[:cores])  # warm-up
        t0 = time.perf_counter()
        done = sum(pool.map(_cpu_worker, jobs))
        t_cpu = time.perf_counter() - t0
    cpu_rate = done / t_cpu  # trials per second (mix of the 8 experiments)
    line = {
        "workload": "acceptance criterion 8 set: B=256 U=16 C=8 16-QAM, SNR 9.5/11/12.5 dB, "
                    f"{args.trials} trials, MRC/ZF/L-MMSE/LAMA x PD/FD (seed 1)",
        "trials_total": n_exp_trials,
        "gpu_seconds": t_gpu, "gpu_trials_per_s": n_exp_trials / t_gpu,
        "run_experiment_seconds_incl_predictions": t_run,
        "host_draw_seconds_shared": t_draw,
        "cpu_trials_per_s": cpu_rate, "cpu_cores": cores,
        "cpu_sample": f"{done} trials (SNR 11 dB, all 8 experiments) through the oracle port of the "
                      f"reference path, {t_cpu:.1f} s on {cores} processes",
        "cpu_seconds_extrapolated": n_exp_trials / cpu_rate,
        "speedup_vs_cpu": (n_exp_trials / t_gpu) / cpu_rate,
        "orderings_ok": bool(ok),
        "ser": {f"{k}-{a}": [round(p.ser, 5) for p in results[k, a].points] for k in KINDS for a in ARCHS},
        "ser_predicted": {f"{k}-{a}": [round(p.ser_predicted, 5) for p in results[k, a].points]
                          for k in KINDS for a in ARCHS},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
