"""Print the analytic cost/memory table (costmodel.py) for the BASELINE configurations.

    python tools/cost_report.py [--fwd-tflops F] [--bwd-tflops B] [--link-gbps L]

Kernel rates default to the round-1 single-GPU measurements (profiles/README.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00611_b200 import costmodel as cm  # noqa: E402
from paper_2407_00611_b200.scheduler import candidates  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fwd-tflops", type=float, default=853.0)
    ap.add_argument("--bwd-tflops", type=float, default=1020.0)
    ap.add_argument("--link-gbps", type=float, default=700.0)
    a = ap.parse_args()
    rows = [("gpt", N, 32, 128, True, P) for P in (1, 2, 4, 8) for N in (max(32768, 16384 * P),)]
    rows += [("gpt", N, 32, 128, True, 8) for N in (16384 * 8 * 2, 16384 * 8 * 4)]
    rows += [("dit", 65536, 16, 72, False, P) for P in (1, 8)]
    print(f"{'workload':8} {'N':>7} {'P':>2} {'C':>2} {'reg':5} {'R':>2} {'recv MiB':>9} {'ws GiB':>7} {'ws/A':>6} "
          f"{'pred ms':>8} {'exposed':>8} {'TF/s/GPU':>9}")
    for wl, N, h, d, causal, P in rows:
        for C in candidates(P):
            pr = cm.predict(P, C, N, h, d, causal, a.fwd_tflops, a.bwd_tflops, a.link_gbps)
            mem = cm.memory(P, C, N, h, d, causal)
            ff, fb = cm.flops(N, h, d, causal)
            print(f"{wl:8} {N:7d} {P:2d} {C:2d} {pr['regime']:5} {pr['R']:2d} {pr['recv_bytes_max'] / 2**20:9.0f} "
                  f"{mem['workspace_bytes'] / 2**30:7.2f} {mem['workspace_over_A']:6.1f} {pr['total_ms']:8.2f} "
                  f"{pr['exposed_comm_frac']:8.3f} {(ff + fb) / P / pr['total_ms'] / 1e9:9.0f}")


if __name__ == "__main__":
    main()
