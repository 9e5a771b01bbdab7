#!/usr/bin/env python
"""Per-rank cost of the strong-scaling (batch-1 query-split) bench at N = 1/2/4/8, simulated on ONE
GPU: rank 0's share of config 2 runs alone, torch.distributed not initialised, so the Q^c gather and
the output gather degenerate to local copies (no NCCL time).  Prints one JSON line per N with the
per-chunk ms and the per-stage device-time shares -- what bounds the per-rank chunk latency as N
grows (perf experiment; the real N > 1 numbers are the driver's scaling run)."""
import argparse
import contextlib
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ns = [int(x) for x in os.environ.get("NS", "1,2,4,8").split(",")]
    for n in ns:
        args = argparse.Namespace(gpus=n, steps=int(os.environ.get("STEPS", "30")), warmup=3, impl="ours",
                                  k_top=bench.GEOM["k_top"], scaling="strong", no_e2e=True, no_cpu=True, out=None)
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            bench.run_ours(args, 0, n, 0)
        line = [l for l in buf.getvalue().splitlines() if l.startswith("{")][-1]
        j = json.loads(line)
        print(json.dumps({"n": n, "rank0_ms_per_chunk": j["ms_per_step"], "k3_ms": j["roofline"]["avg_launch_ms"],
                          "k3_frac": j["roofline"]["frac"], "stage_share": j.get("stage_share_of_step"),
                          "gpu_launches": j.get("gpu_launches")}), flush=True)


if __name__ == "__main__":
    main()
