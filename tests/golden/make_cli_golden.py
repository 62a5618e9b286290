"""`map` command fixtures produced by the reference CLI itself (SURVEY §8(f) #4 pins).

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: an INI run configuration, a float32 and an int16 WAV
recording of a delayed common source, the reference `cmd_precompute` caches for
sspi and conv, and the reference `cmd_map` CSVs (with a --truth location), plus
cli_golden.npz with the reference `load_audio` output of both recordings.
"""

from __future__ import annotations

import os
import sys

import numpy as np
from scipy.io import wavfile

sys.path.insert(0, "/root/reference/pkg/src")

from srpmap import cli  # noqa: E402
from srpmap.config import MethodSpec, load_config  # noqa: E402
from srpmap.frontend import load_audio  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")

CONFIG = """[scenario]
mode = nf
room = 4 4 3

[array]
kind = positions
positions = 0.45 0.50 0; 0.58 0.47 0; 0.52 0.62 0; 0.40 0.60 0
speed_of_sound = 343

[grid]
origin = 0 0 0
extents = 1 1 0
resolution = 0.1

[pipeline]
frame_len = 256
sample_rate = 16000
weighting = phat
n_aux = 2
"""


def main():
    os.makedirs(OUT, exist_ok=True)
    cfg_path = os.path.join(OUT, "run.ini")
    with open(cfg_path, "w") as fh:
        fh.write(CONFIG)
    cfg = load_config(cfg_path)
    rng = np.random.default_rng(2306)
    m, nf = cfg.scenario.array.num_mics, 12
    n = (nf - 1) * cfg.frame.hop + cfg.frame.frame_len + 37          # a ragged tail (not a full frame)
    src = rng.standard_normal(n + 16)
    sig = 0.2 * rng.standard_normal((m, n))
    for ch, d in enumerate((0, 3, 5, 2)):
        sig[ch] += src[d:d + n]
    sig *= 0.25
    wav32 = os.path.join(OUT, "scene_f32.wav")
    wavfile.write(wav32, 16000, sig.T.astype(np.float32))
    wav16 = os.path.join(OUT, "scene_i16.wav")
    wavfile.write(wav16, 16000, np.round(sig.T * 32767).clip(-32768, 32767).astype(np.int16))
    golden = {}
    for tag, path in (("f32", wav32), ("i16", wav16)):
        x, rate = load_audio(path)
        golden[f"audio_{tag}"] = x
        golden[f"rate_{tag}"] = np.float64(rate)
    truth = "0.5 0.5 0"
    for kind, extra in (("sspi", dict(sparsity="2jp")), ("conv", {})):
        method = MethodSpec(name=kind, path="ifft", **extra)
        cfg_k = cli.RunConfig(scenario=cfg.scenario, frame=cfg.frame, weighting=cfg.weighting,
                              n_aux=cfg.n_aux, method=method) if hasattr(cli, "RunConfig") else None
        if cfg_k is None:
            from srpmap.config import RunConfig
            cfg_k = RunConfig(scenario=cfg.scenario, frame=cfg.frame, weighting=cfg.weighting,
                              n_aux=cfg.n_aux, method=method)
        cache = os.path.join(OUT, f"{kind}.srpm")
        cli.cmd_precompute(cfg_k, cache)
        for tag, path in (("f32", wav32), ("i16", wav16)):
            out = os.path.join(OUT, f"map_{kind}_{tag}.csv")
            cli.cmd_map(cfg_k, cache, path, out, truth)
    np.savez_compressed(os.path.join(HERE, "cli_golden.npz"), **golden)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
