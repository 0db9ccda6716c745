"""Runs AC5's disturbance scenario once on 2 ranks with ICCL_DEBUG=1 and
prints both ranks' logs (the pytest run keeps them in a temp dir)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["ICCL_DEBUG"] = "1"
import gpu_scenarios as sc  # noqa: E402
from gpu_helpers import run_ranks  # noqa: E402



def competing():
    import numpy as np
    MiB = 1 << 20
    os.environ["ICCL_DEBUG"] = "0"
    with tempfile.TemporaryDirectory() as d:
        res = run_ranks(2, sc.monitor_competing, d, nchunks=384, chunk=16 * MiB, comp_bytes=2048 * MiB,
                        delay_us=2000, config=dict(chunk_bytes=16 * MiB, monitor_enabled=True, window=1024))
        t1, t2 = res[0]["t1"], res[0]["t2"]
        dur = (t2 - t1) / 1e3
        print("competing: records", len(dur), "span us", (t2[-1] - t1[0]) / 1e3)
        print("durations us (every 8th):", np.round(dur[::8], 1).tolist())


def main():
    MiB = 1 << 20
    with tempfile.TemporaryDirectory() as d:
        try:
            res = run_ranks(2, sc.monitor_accuracy, d, nchunks=128, chunk=16 * MiB, stall_chunk=64, up_us=200_000,
                            config=dict(chunk_bytes=16 * MiB, monitor_enabled=True, delta_us=5_000_000, window=1024))
            print("switches", [r["switches"] for r in res], [r["switch_desc"] for r in res])
            for r in res:
                if len(r["t2"]):
                    import numpy as np
                    du = r["t2"] - r["t1"]
                    print("records", len(du), "dur min/med/max ns", du.min(), int(np.median(du)), du.max(),
                          "span us", (r["t2"][-1] - r["t1"][0]) / 1e3)
        finally:
            for r in range(2):
                p = os.path.join(d, f"rank{r}.log")
                if os.path.exists(p):
                    lines = open(p).read().splitlines()
                    print(f"---- rank {r}: {len(lines)} lines")
                    keep = [ln for ln in lines if "fault" in ln or "gate" in ln or "switch" in ln or "issue" in ln
                            or "posted" in ln or "Error" in ln or "armed pair" in ln]
                    print("\n".join(keep[:200]))


if __name__ == "__main__":
    main()
    competing()
