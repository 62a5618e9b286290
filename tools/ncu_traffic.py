"""Per-launch DRAM traffic of the hot-path kernels from `ncu --set full` raw exports.

    python tools/ncu_traffic.py cfg2:sspi:profiles/r1_full_cfg2_sspi_raw.csv ... > profiles/traffic.json

Each argument is workload:variant:csv.  Output: {workload: {variant: {kernel: bytes}}}
with kernels keyed the way bench.py names the dominant kernel (`frontend`,
`<variant>_map`, `fused` for the one-kernel SSPI chain, `srp_map_tc` for the stored-operator tensor-core map, `srp_map_tdoa`
for the on-chip-steering one; `<variant>_factor` for the low-rank factor product); the
value is dram__bytes_read.sum + dram__bytes_write.sum averaged over that kernel's launches.
"""

import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def key_of(name: str, variant: str):
    if "frontend_map_kernel" in name or "frontend_sspi" in name:
        return "fused"
    if "untile" in name:
        return f"{variant}_untile"
    if "gather_pair_kernel" in name:      # bench.py's name of the CTA-pair gathered-window kernels
        return "gather_pair_kernel<PairF16>" if "PairF16" in name else "gather_pair_kernel<PairTf32>"
    if "gather_tc" in name:
        return f"{variant}_map"
    if "frontend" in name:
        return "frontend"
    if "conv_gen_chunked_kernel" in name:
        targs = name.split("conv_gen_chunked_kernel<", 1)[1].split(">", 1)[0].replace(" ", "")
        return "srp_map_tdoa" if targs.endswith(("true", "1")) else "srp_map_tc"   # <SPLIT, GEN>
    if "sspi" in name or "interp_tc" in name:
        return f"{variant}_map"
    if "lowrank_out" in name:
        return f"{variant}_map"
    if "splitk" in name and variant in ("conv", "conv_h"):
        return "srp_map_splitk_reduce"
    if "gemm_nt" in name or "splitk" in name or "split_bf16" in name:
        return f"{variant}_factor"
    return None


def main(args):
    out = {}
    if args and args[0].startswith("--merge="):      # keep the entries of an existing traffic.json
        with open(args[0].split("=", 1)[1]) as f:
            out = json.load(f)
        args = args[1:]
    for a in args:
        workload, variant, path = a.split(":", 2)
        with open(path) as f:
            rows = list(csv.reader(f))
        hdr, units = rows[0], rows[1]
        ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        acc = {}
        for r in rows[2:]:
            k = key_of(r[hdr.index("Kernel Name")], variant)
            if k is None:
                continue
            b = (float(r[ir].replace(",", "")) * UNITS.get(units[ir], 1)
                 + float(r[iw].replace(",", "")) * UNITS.get(units[iw], 1))
            acc.setdefault(k, []).append(b)
        for k, v in acc.items():
            out.setdefault(workload, {}).setdefault(variant, {})[k] = sum(v) / len(v)
        out.setdefault("_sources", {})[f"{workload}:{variant}"] = path
    json.dump(out, sys.stdout, indent=1, sort_keys=True)
    print()


if __name__ == "__main__":
    main(sys.argv[1:])
