"""Synthetic scenes and the `sweep` command on the B200 engine.

The reference's error/accuracy sweep (cli.py:287-398) renders random source placements
in a shoebox room (simulate.py), maps every frame with the conventional SRP and with each
configured LR / SI / SLRI / SSPI operator, and writes one CSV row per operator:
relative cost, operator error, map-error percentiles and mean localisation accuracy.
Here the frame loop runs batched on the GPU:

* rendering: source placement, image sources, fractional-delay kernels, pink noise and
  the SNR scaling follow simulate.py on the host (same seeded generator sequence); the
  room-response convolution -- the expensive part, microphones x images x samples x 64
  taps -- is `srpgpu_render_images` (float64);
* every placement's frames go through the fused frontend (`gcc_frames`,
  `frames_to_samples`) and the batched map kernels; the conventional reference maps
  use the fp32 SIMT GEMM (`precision="fp32"`);
* cost, operator errors (eps_h), SVDs and sparse fits are host float64 as in the
  reference; map errors and argmax scores are computed from the GPU maps.

`python -m paper_2306_08514_b200.sweep run.ini out.csv` writes the reference's CSV.
"""

from __future__ import annotations

import configparser
import csv
import math
import sys
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _native as nat
from . import frontend as fe
from . import maps, operators, sampling, scene
from .batch import FF_THRESHOLD, NF_THRESHOLD, fmt, load_audio, loc_accuracy, loc_error, read_run_config
from .errors import ConfigError

TAPS = 64                          # simulate.py:26 fractional-delay filter length
SWEEP_HEADER = ["method", "param_name", "param_value", "c_rel", "eps_h_db",
                "eps_z_db_p10", "eps_z_db_p50", "eps_z_db_p90", "rho_s_mean"]


# ----------------------------------------------------------------- configuration

@dataclass(frozen=True)
class Scenario:
    """The [scenario] section (simulate.py:31-76 ScenarioConfig, config.py:192-208)."""

    mode: str
    room: np.ndarray
    array: object
    grid: object
    sample_rate: float
    source: str = "pink"
    reflection_order: int = 0
    absorption: np.ndarray = None
    snr_db: float = math.inf
    num_placements: int = 1
    frames_per_placement: int = 1
    seed: int = 0
    placement: str = "random"
    ff_range: tuple = (2.5, 3.0)


@dataclass(frozen=True)
class SweepConfig:
    run: object                    # batch.RunScene (array, grid, frame, weighting, n_aux)
    scenario: Scenario
    methods: tuple
    ranks: tuple
    sparsities: tuple
    path: str = "auto"


def read_sweep_config(path: str) -> SweepConfig:
    """A reference INI run configuration with a [sweep] section (config.py:159-240)."""
    run = read_run_config(path)
    cp = configparser.ConfigParser(inline_comment_prefixes=(";", "#"))
    cp.read(path)
    sc = cp["scenario"]
    snr_text = sc.get("snr_db", "inf")
    absorption = np.array([float(t) for t in sc.get("absorption", "0.5").split()])
    absorption = np.broadcast_to(absorption if absorption.size > 1 else absorption[0], (6,)).astype(float)
    if np.any(absorption < 0) or np.any(absorption > 1):
        raise ConfigError("absorption must lie in [0, 1]")
    kw = {}
    if "ff_range" in sc:
        kw["ff_range"] = tuple(float(t) for t in sc["ff_range"].split())
    placement = sc.get("placement", "random")
    if placement not in ("random", "on_grid"):
        raise ConfigError(f"unknown placement policy {placement!r}")
    scen = Scenario(mode=run.mode, room=np.asarray(run.room, dtype=float), array=run.array, grid=run.grid,
                    sample_rate=run.frame.sample_rate, source=sc.get("source", "pink"),
                    reflection_order=int(sc.get("reflection_order", "0")), absorption=absorption,
                    snr_db=math.inf if snr_text in ("inf", "+inf") else float(snr_text),
                    num_placements=int(sc.get("num_placements", "1")),
                    frames_per_placement=int(sc.get("frames_per_placement", "1")),
                    seed=int(sc.get("seed", "0")), placement=placement, **kw)
    if "sweep" not in cp:
        raise ConfigError("sweep needs a [sweep] section")
    sw = cp["sweep"]
    methods = tuple(sw.get("methods", "lr slri sspi").split())
    for m in methods:
        if m not in ("lr", "si", "slri", "sspi"):
            raise ConfigError(f"sweep.methods must be lr / si / slri / sspi, got {m!r}")
    path_token = cp["method"].get("path", "auto") if "method" in cp else "auto"
    return SweepConfig(run=run, scenario=scen, methods=methods, ranks=tuple(sw.get("ranks", "").split()),
                       sparsities=tuple(sw.get("sparsities", "").split()), path=path_token)


# ----------------------------------------------------------------- scene synthesis

def _inside(p, room, margin: float = 1e-6) -> bool:
    return bool(np.all(p > margin) and np.all(p < room - margin))


def place_sources(sc: Scenario) -> np.ndarray:
    """True source positions (num_placements, 3) (simulate.py:80-121): seeded by
    (seed, 0); NF uniform in the grid's bounding box, FF along a grid or random polar-cap
    direction at a distance in ff_range from the array centre, inside the room."""
    rng = np.random.default_rng([sc.seed, 0])
    out = np.empty((sc.num_placements, 3))
    if sc.mode == "nf":
        pts = sc.grid.points
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        if not (_inside(lo, sc.room) and _inside(hi, sc.room)):
            raise ConfigError("search grid extends outside the room")
        for i in range(sc.num_placements):
            out[i] = pts[rng.integers(len(pts))] if sc.placement == "on_grid" else rng.uniform(lo, hi)
        return out
    centre = sc.array.center
    for i in range(sc.num_placements):
        for _ in range(1000):
            if sc.placement == "on_grid":
                u = sc.grid.points[rng.integers(len(sc.grid.points))]
            else:
                polar = np.deg2rad(rng.uniform(sc.grid.axes[0][0], sc.grid.axes[0][-1]))
                azim = rng.uniform(0.0, 2.0 * np.pi)
                u = np.array([np.sin(polar) * np.cos(azim), np.sin(polar) * np.sin(azim), np.cos(polar)])
            cand = centre - rng.uniform(*sc.ff_range) * u
            if _inside(cand, sc.room):
                out[i] = cand
                break
        else:
            raise ConfigError("could not place a far-field source inside the room")
    return out


def true_location(sc: Scenario, source) -> np.ndarray:
    """Position (NF) or unit propagation direction towards the array (FF) (simulate.py:130-137)."""
    source = np.asarray(source, dtype=float)
    if sc.mode == "nf":
        return source
    d = sc.array.center - source
    return d / np.linalg.norm(d)


def delay_kernel(frac: float) -> np.ndarray:
    """64-tap Hann-windowed sinc delaying by 31 + frac samples (simulate.py:140-150)."""
    u = np.arange(TAPS) - (TAPS // 2 - 1) - frac
    w = 0.5 * (1.0 + np.cos(np.pi * u / (TAPS // 2)))
    w[np.abs(u) >= TAPS // 2] = 0.0
    return np.sinc(u) * w


def pink_noise(rng, n: int) -> np.ndarray:
    """Unit-variance 1/f-power noise from white noise shaped in the rfft domain (simulate.py:153-161)."""
    spec = np.fft.rfft(rng.standard_normal(n))
    f = np.fft.rfftfreq(n)
    spec[0] = 0.0
    spec[1:] /= np.sqrt(f[1:])
    out = np.fft.irfft(spec, n=n)
    return out / np.std(out)


def image_sources(source, room, max_order: int, absorption):
    """Shoebox image sources up to `max_order` reflections (simulate.py:164-205): per axis,
    images at +-x + 2 n L with wall-hit counts; products over the three axes; ordered by
    reflection order, then enumeration order.  Returns (positions, gains, orders)."""
    source = np.asarray(source, dtype=float)
    beta = np.sqrt(1.0 - np.asarray(absorption, dtype=float))
    span = max_order // 2 + 1
    axis_terms = []
    for d in range(3):
        terms = []
        for n in range(-span, span + 1):
            for mirror in (0, 1):
                if mirror == 0:
                    lo_hits = hi_hits = abs(n)
                else:
                    lo_hits, hi_hits = (n - 1, n) if n >= 1 else (1 - n, -n)
                if lo_hits + hi_hits <= max_order:
                    coord = (source[d] if mirror == 0 else -source[d]) + 2 * n * room[d]
                    terms.append((coord, lo_hits + hi_hits, beta[2 * d] ** lo_hits * beta[2 * d + 1] ** hi_hits))
        axis_terms.append(terms)
    pos, gain, order = [], [], []
    for cx, ox, gx in axis_terms[0]:
        for cy, oy, gy in axis_terms[1]:
            for cz, oz, gz in axis_terms[2]:
                if ox + oy + oz <= max_order:
                    pos.append((cx, cy, cz))
                    gain.append(gx * gy * gz)
                    order.append(ox + oy + oz)
    pos, gain, order = np.asarray(pos), np.asarray(gain), np.asarray(order)
    idx = np.lexsort((np.arange(order.shape[0]), order))
    return pos[idx], gain[idx], order[idx]


def _dry_signal(sc: Scenario, rng, n: int) -> np.ndarray:
    if sc.source == "pink":
        return pink_noise(rng, n)
    data, rate = load_audio(sc.source)
    if abs(rate - sc.sample_rate) > 1e-9:
        raise ConfigError(f"source file rate {rate} Hz does not match scenario rate {sc.sample_rate} Hz")
    if data.shape[1] < n:
        raise ConfigError("source file too short for the requested render")
    return np.asarray(data[0][:n], dtype=float)


def room_response(sc: Scenario, source, dry: np.ndarray, device: bool = True):
    """(direct, reverb) (M, N) float64: the image-source sum of 64-tap fractional-delay
    filters of `dry` (simulate.py:238-254), on the GPU (`srpgpu_render_images`) or, with
    device=False, on the host with np.convolve (the reference's own arithmetic)."""
    mics = sc.array.positions
    fs, c = sc.sample_rate, sc.array.speed_of_sound
    n = dry.shape[0]
    pos, gain, order = image_sources(source, sc.room, sc.reflection_order, sc.absorption)
    m_count, i_count = mics.shape[0], pos.shape[0]
    start = np.empty((m_count, i_count), dtype=np.int64)
    g = np.empty((m_count, i_count))
    taps = np.empty((m_count, i_count, TAPS))
    for m in range(m_count):
        for i in range(i_count):
            dist = float(np.linalg.norm(mics[m] - pos[i]))
            delay = dist * fs / c
            base = int(np.floor(delay))
            taps[m, i] = delay_kernel(delay - base)
            g[m, i] = gain[i] / max(dist, 1e-6)
            start[m, i] = base - (TAPS // 2 - 1)
    if not device:
        direct, reverb = np.zeros((m_count, n)), np.zeros((m_count, n))
        for m in range(m_count):
            for i in range(i_count):
                r = np.convolve(dry, taps[m, i]) * g[m, i]
                s0 = int(start[m, i])
                lo, hi = max(s0, 0), min(s0 + r.shape[0], n)
                if hi > lo:
                    (direct if order[i] == 0 else reverb)[m, lo:hi] += r[lo - s0:hi - s0]
        return direct, reverb
    d = dev.device()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(d)
    dry_d, start_d, g_d, taps_d = t(dry, np.float64), t(start, np.int64), t(g, np.float64), t(taps, np.float64)
    is_direct = t((order == 0).astype(np.int32), np.int32)
    direct = torch.empty((m_count, n), dtype=torch.float64, device=d)
    reverb = torch.empty((m_count, n), dtype=torch.float64, device=d)
    nat.call("srpgpu_render_images", dev.ptr(dry_d), n, m_count, i_count, dev.ptr(start_d), dev.ptr(g_d),
             dev.ptr(taps_d), dev.ptr(is_direct), dev.ptr(direct), dev.ptr(reverb), dev.stream_ptr())
    return direct.cpu().numpy(), reverb.cpu().numpy()


def synthesize(sc: Scenario, source, num_samples: int, seed_offset: int = 0, device: bool = True) -> np.ndarray:
    """(M, num_samples) microphone signals of one placement (simulate.py:208-265): dry
    source from the (seed, 1 + placement) generator, room response, then independent pink
    channel noise at snr_db relative to the direct-path power."""
    source = np.asarray(source, dtype=float)
    if not _inside(source, sc.room):
        raise ConfigError(f"source {source} outside the room")
    if np.min(np.linalg.norm(sc.array.positions - source[None, :], axis=1)) < 1e-9:
        raise ConfigError("source coincides with a microphone")
    rng = np.random.default_rng([sc.seed, 1 + seed_offset])
    dry = _dry_signal(sc, rng, num_samples)
    direct, reverb = room_response(sc, source, dry, device)
    mix = direct + reverb
    if math.isfinite(sc.snr_db):
        p_direct = float(np.mean(direct ** 2))
        if p_direct == 0.0:
            raise ConfigError("direct path has zero power; cannot set an SNR")
        noise = np.stack([pink_noise(rng, num_samples) for _ in range(sc.array.num_mics)])
        mix = mix + math.sqrt(p_direct * 10.0 ** (-sc.snr_db / 10.0) / float(np.mean(noise ** 2))) * noise
    return mix


def render_for_frames(sc: Scenario, frame, source, seed_offset: int = 0, device: bool = True) -> np.ndarray:
    """Signal for frames_per_placement frames after one frame length of lead-in
    (simulate.py:268-280)."""
    if abs(frame.sample_rate - sc.sample_rate) > 1e-9:
        raise ConfigError("frame spec and scenario sample rates disagree")
    needed = frame.frame_len + frame.hop * (sc.frames_per_placement - 1)
    return synthesize(sc, source, needed + frame.frame_len, seed_offset, device)[:, frame.frame_len:]


# ----------------------------------------------------------------- cost / error metrics

def sampling_cost(num_pairs: int, num_bins: int, total_samples: float, path: str = "auto"):
    """Multiplications of the TD-GCC sampling step and the path taken (metrics.py:64-79)."""
    k = num_bins + 1
    by_matrix = 2.0 * total_samples * num_bins
    by_ifft = 8.0 * num_pairs * k * math.log2(2 * k)
    if path == "matrix":
        return by_matrix
    if path == "ifft":
        return by_ifft
    if path != "auto":
        raise ValueError(f"unknown sampling path {path!r}")
    return by_ifft if by_ifft < by_matrix else by_matrix


def relative_cost(method: str, j: int, p: int, b: int, total_samples=None, rank=None, keep=None,
                  path: str = "auto") -> float:
    """Multiplications relative to conventional SRP (metrics.py:82-125)."""
    base = 2 * j * p * b
    if method == "conv":
        total = float(base)
    elif method == "lr":
        total = 2.0 * j * rank + 4.0 * rank * p * b
    else:
        samp = sampling_cost(p, b, total_samples, path)
        total = {"si": lambda: j * total_samples + samp,
                 "slri": lambda: j * rank + rank * total_samples + samp,
                 "sspi": lambda: keep + samp}[method]()
    return float(total) / base


def _db(diff_sq: float, ref_sq: float) -> float:
    if ref_sq == 0.0:
        raise ValueError("reference has zero norm; relative error undefined")
    return -math.inf if diff_sq == 0.0 else 10.0 * math.log10(diff_sq / ref_sq)


def matrix_error(approx, reference) -> float:
    """Relative Frobenius error in dB, -inf when equal (metrics.py:128-149)."""
    a, r = np.asarray(approx), np.asarray(reference)
    return _db(float(np.sum(np.abs(a - r) ** 2)), float(np.sum(np.abs(r) ** 2)))


def svd_tail_db(s: np.ndarray, rank: int) -> float:
    """Rank-R truncation error from the singular values (metrics.py:152-161)."""
    s = np.asarray(s, dtype=float)
    return _db(float(np.sum(s[rank:] ** 2)), float(np.sum(s ** 2)))


def percentile(values, q: float) -> float:
    """Linear-interpolation percentile that tolerates -inf entries (cli.py:287-295)."""
    v = np.sort(np.asarray(values, dtype=float))
    pos = (v.size - 1) * q / 100.0
    lo, hi = int(np.floor(pos)), int(np.ceil(pos))
    a, b = float(v[lo]), float(v[hi])
    if lo == hi or a == b or np.isneginf(a):
        return a
    return a + (b - a) * (pos - lo)


def dense_sampling_matrix(spec, half_len: int) -> np.ndarray:
    """Block-diagonal single-sided sampling matrix (S, P*B) (sampling.py:179-197)."""
    bins = half_len - 1
    off = sampling.spec_offsets(spec)
    out = np.zeros((int(off[-1]), spec.num_pairs * bins), dtype=np.complex128)
    k = np.arange(1, half_len)
    for p in range(spec.num_pairs):
        c = int(spec.counts[p])
        lags = np.concatenate([np.arange(0, c + 1), np.arange(-c, 0)])
        out[off[p]:off[p + 1], p * bins:(p + 1) * bins] = np.exp(1j * np.pi * np.outer(lags, k) / half_len)
    return out


def _resolve_rank(token: str, full: int) -> int:
    if token == "full":
        return full
    rank = int(token)
    if not 1 <= rank <= full:
        raise ConfigError(f"rank {rank} outside [1, {full}]")
    return rank


# ----------------------------------------------------------------- the sweep

def run_sweep(cfg: SweepConfig, device_render: bool = True) -> list:
    """CSV rows of the reference sweep (cli.py:309-388), maps on the GPU."""
    run, sc = cfg.run, cfg.scenario
    frame, grid = run.frame, run.grid
    pairs = scene.enumerate_pairs(run.array)
    tdoa = scene.tdoa_table(run.array, pairs, grid)
    spec = sampling.sample_spec(tdoa, frame, run.n_aux)
    j, p, b = grid.num_points, pairs.num_pairs, frame.num_bins
    s_tot = int(sampling.spec_offsets(spec)[-1])
    srp = operators.build_srp_matrix(tdoa, frame, max_bytes=1 << 36)
    interp = operators.build_interp_matrix(tdoa, spec, frame, max_bytes=1 << 36)
    samp_dense = dense_sampling_matrix(spec, frame.half_len)

    # every placement's frames through the GPU frontend, concatenated
    psi, xi, truths = [], [], []
    fpp = sc.frames_per_placement
    for i, pos in enumerate(place_sources(sc)):
        sig = render_for_frames(sc, frame, pos, seed_offset=i, device=device_render)
        x = torch.from_numpy(np.ascontiguousarray(sig, dtype=np.float32)).to(dev.device())
        psi.append(fe.gcc_frames(x, frame, pairs, range(fpp), run.weighting).values)
        xi.append(sampling.frames_to_samples(x, frame, pairs, spec, range(fpp), run.weighting).values)
        truths += [true_location(sc, pos)] * fpp
    psi, xi = torch.cat(psi), torch.cat(xi)
    gcc = fe.FdGcc(psi, p, b, run.weighting)
    samples = sampling.TdGccSamples(xi.contiguous(), spec)
    z_ref = maps.srp_map_exact(srp, gcc, precision="fp32").double()
    ref_sq = (z_ref * z_ref).sum(dim=1)
    if bool((ref_sq == 0).any()):
        raise ValueError("reference has zero norm; relative error undefined")
    thr = NF_THRESHOLD if grid.mode == "nf" else FF_THRESHOLD

    def score(idx: np.ndarray) -> float:
        return float(np.mean([loc_accuracy(loc_error(grid.points[k], t, grid.mode), thr)
                              for k, t in zip(idx, truths)]))

    rows = []

    def add(method, pname, pval, c_rel, eps_h, z):
        # per-frame map error (metrics.map_error) on the device in float64: one reduction per
        # operator instead of a host loop over frames
        z = z.double()
        d = ((z - z_ref) ** 2).sum(dim=1)
        errs = torch.where(d == 0, torch.full_like(d, -math.inf), 10.0 * torch.log10(d / ref_sq))
        idx = torch.argmax(z, dim=1).cpu().numpy()         # first maximum, as np.argmax
        errs = errs.cpu().numpy()
        rows.append([method, pname, str(pval), fmt(c_rel), fmt(eps_h)]
                    + [fmt(percentile(errs, q)) for q in (10, 50, 90)] + [fmt(score(idx))])

    add("conv", "", "", relative_cost("conv", j, p, b), -math.inf, z_ref)
    if "si" in cfg.methods:
        add("si", "", "", relative_cost("si", j, p, b, s_tot, path=cfg.path),
            matrix_error(interp.matrix @ samp_dense, srp.matrix), maps.si_map(interp, samples))
    if "lr" in cfg.methods and cfg.ranks:
        u, s, vt = np.linalg.svd(srp.matrix, full_matrices=False)
        for tok in cfg.ranks:
            r = _resolve_rank(tok, s.shape[0])
            op = operators.low_rank_srp_from_svd(u, s, vt, r)
            add("lr", "rank", r, relative_cost("lr", j, p, b, rank=r), svd_tail_db(s, r), maps.lr_map(op, gcc))
    if "slri" in cfg.methods and cfg.ranks:
        u, s, vt = np.linalg.svd(interp.matrix, full_matrices=False)
        for tok in cfg.ranks:
            r = _resolve_rank(tok, s.shape[0])
            op = operators.low_rank_interp_from_svd(u, s, vt, r)
            add("slri", "rank", r, relative_cost("slri", j, p, b, s_tot, rank=r, path=cfg.path),
                matrix_error(op.to_dense() @ samp_dense, srp.matrix), maps.slri_map(op, samples))
    if "sspi" in cfg.methods and cfg.sparsities:
        for tok in cfg.sparsities:
            keep = operators.resolve_sparsity(tok, j, p, interp.matrix.size)
            op = operators.truncate_sparse(interp, keep)
            add("sspi", "keep", keep, relative_cost("sspi", j, p, b, s_tot, keep=keep, path=cfg.path),
                matrix_error(op.to_dense() @ samp_dense, srp.matrix), maps.sspi_map(op, samples))
    return rows


def cmd_sweep(cfg: SweepConfig, out_path: str) -> None:
    rows = run_sweep(cfg)
    with open(out_path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SWEEP_HEADER)
        w.writerows(rows)
    print(f"sweep CSV with {len(rows)} rows written to {out_path}")


if __name__ == "__main__":
    if len(sys.argv) != 3:
        sys.exit("usage: python -m paper_2306_08514_b200.sweep run.ini out.csv")
    cmd_sweep(read_sweep_config(sys.argv[1]), sys.argv[2])
