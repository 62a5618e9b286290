"""`sweep` command and scene-rendering fixtures produced by the reference itself
(SURVEY §8(f) #4 pins).

Run in the build container (where /root/reference exists):

    python tests/golden/make_sweep_golden.py

Writes tests/golden/sweep/: two INI run configurations (a reverberant near-field room
with noise, an anechoic far-field circular array) and the reference `cmd_sweep` CSV of
each, plus sweep_golden.npz with the reference `place_sources`, `image_sources` and
`render_for_frames` outputs of both scenarios.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from srpmap import cli, simulate  # noqa: E402
from srpmap.config import load_config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "sweep")

CONFIGS = {
    "nf_room": """[scenario]
mode = nf
room = 4 4 3
reflection_order = 2
absorption = 0.4
snr_db = 20
num_placements = 3
frames_per_placement = 3
seed = 7
placement = random

[array]
kind = positions
positions = 1.80 1.85 1.0; 2.15 1.80 1.0; 2.20 2.20 1.0; 1.85 2.15 1.0
speed_of_sound = 343

[grid]
origin = 1 1 1
extents = 2 2 0
resolution = 0.25

[pipeline]
frame_len = 512
sample_rate = 16000
weighting = phat
n_aux = 2

[sweep]
methods = lr si slri sspi
ranks = 1 4 full
sparsities = 1jp 2jp all
""",
    "ff_uca": """[scenario]
mode = ff
room = 6 6 4
reflection_order = 0
snr_db = inf
num_placements = 2
frames_per_placement = 2
seed = 3
placement = on_grid
ff_range = 2.5 2.8

[array]
kind = circular
center = 3 3 2
radius = 0.05
count = 6
speed_of_sound = 343

[grid]
polar_deg = 90 180
azimuth_deg = 0 360
resolution_deg = 30

[pipeline]
frame_len = 256
sample_rate = 16000
weighting = phat

[sweep]
methods = slri sspi
ranks = 2 full
sparsities = 0.5jp 1jp
""",
}


def main():
    os.makedirs(OUT, exist_ok=True)
    arrays = {}
    for name, text in CONFIGS.items():
        ini = os.path.join(OUT, f"{name}.ini")
        with open(ini, "w") as f:
            f.write(text)
        cfg = load_config(ini)
        scen = cfg.scenario
        pos = simulate.place_sources(scen)
        arrays[f"{name}_sources"] = pos
        img, gains, orders = simulate.image_sources(pos[0], scen.room, scen.reflection_order, scen.absorption)
        arrays[f"{name}_img_pos"], arrays[f"{name}_img_gain"], arrays[f"{name}_img_order"] = img, gains, orders
        for i, p in enumerate(pos):
            arrays[f"{name}_render_{i}"] = simulate.render_for_frames(scen, cfg.frame, p, seed_offset=i)
            arrays[f"{name}_truth_{i}"] = simulate.true_location(scen, p)
        cli.cmd_sweep(cfg, os.path.join(OUT, f"{name}_sweep.csv"))
    np.savez_compressed(os.path.join(HERE, "sweep_golden.npz"), **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
