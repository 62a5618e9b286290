"""Wall time of the sweep command: this engine (GPU maps, GPU room rendering) and, where
/root/reference exists (the build container), the reference cli.run_sweep on the host.

    python tools/bench_sweep.py tools/configs/sweep_cfg1.ini [--reference]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ini = sys.argv[1]
    out = {"config": ini}
    if "--reference" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from srpmap import cli
        from srpmap.config import load_config
        t = time.perf_counter()
        rows = cli.run_sweep(load_config(ini))
        out.update(reference_s=time.perf_counter() - t, reference_rows=len(rows), host_cores=os.cpu_count())
    else:
        import torch
        from paper_2306_08514_b200 import sweep
        cfg = sweep.read_sweep_config(ini)
        sweep.run_sweep(cfg)                      # warm-up: library load, kernel attributes
        torch.cuda.synchronize()
        t = time.perf_counter()
        rows = sweep.run_sweep(cfg)
        torch.cuda.synchronize()
        out.update(engine_s=time.perf_counter() - t, rows=len(rows))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
