"""Summarise an ncu --set full report into profiles/ (json + markdown).

    python tools/ncu_summary.py r01 gpurun_out/prof_a.ncu-rep gpurun_out/prof_b.ncu-rep ...
"""
import csv
import io
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9}


def _key(short: str) -> str:
    """Stable key per kernel: bench.py reads fuse_haar_b6 / fuse_daub4_b6."""
    short = short.replace("wf::", "")
    if short.startswith("fuse_haar_kernel<float"):
        return "fuse_haar_b" + short.split(",")[2].strip()
    if short.startswith("fuse_d4_tma_kernel<float"):
        return "fuse_daub4_b" + short.split(",")[1].strip()
    if short.startswith("quality_split_kernel<"):  # <NB, FUSE>: bench.py reads quality_split_kernel_6
        nb, *fuse = [t.strip() for t in short.split("<")[1].rstrip(">").split(",")]
        return "quality_split_kernel_" + nb + ("_fused" if fuse and fuse[0] not in ("0", "false") else "")
    if short.startswith("fuse_d4_u8x8_kernel<"):  # <NB, NCW, MINB, CVT, EXACT>: v3 = EXACT
        args = [t.strip() for t in short.split("<")[1].rstrip(">").split(",")]
        v2 = len(args) > 4 and args[4] in ("0", "false")
        return "fuse_d4_u8x8_kernel_" + args[0] + ("_v2" if v2 else "")
    if short.startswith("quality_tile64_kernel<"):
        return "quality_tile64_kernel_" + short.split("<")[1].rstrip(">").strip()
    if short.startswith("quality_tile_kernel<"):
        return "quality_tile_kernel_" + short.split("<")[1].rstrip(">").strip()
    return "".join(c if c.isalnum() else "_" for c in short.replace("wf::", "")).strip("_")


def main(reps, tag):
    """Entries of the given reports replace same-key entries of the existing
    profiles/ncu_summary.json; the markdown lists every entry."""
    jp = ROOT / "profiles" / "ncu_summary.json"
    out = json.loads(jp.read_text()) if jp.exists() else {}
    md = [f"# ncu --set full summary ({tag})", "",
                   "Captured with `ncu --set full --clock-control none --import-source on`, one "
                   "launch per kernel after warm-up (tools/profile_once.py, profile_u8.py, "
                   "profile_qnr.py). DRAM % is against ncu's own peak.", "",
                   "| kernel | duration | DRAM read | DRAM write | DRAM % of ncu peak | "
                   "SM % | regs | warps active % | issue IPC | report |",
                   "|---|---|---|---|---|---|---|---|---|---|"]
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        for r in data:
            name = r[hdr.index("Kernel Name")]
            rec = {}
            for k in KEYS + ["sm__inst_executed.avg.per_cycle_active"]:
                if k in hdr:
                    i = hdr.index(k)
                    v = float(r[i].replace(",", "")) if r[i] else None
                    rec[k] = v * SCALE.get(units[i], 1) if v is not None else None
            short = name.split("(")[0].replace("void ", "")
            rec["dram_bytes"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
            rec["kernel"] = short
            rec["report"] = os.path.basename(rep)
            out[_key(short)] = rec
    for rec in out.values():
        md.append(f"| `{rec['kernel']}` | {rec['gpu__time_duration.sum'] * 1e3:.3f} ms | "
                  f"{rec['dram__bytes_read.sum'] / 1e9:.3f} GB | "
                  f"{rec['dram__bytes_write.sum'] / 1e9:.3f} GB | "
                  f"{rec['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                  f"{rec['sm__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                  f"{rec['launch__registers_per_thread']:.0f} | "
                  f"{rec['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                  f"{rec.get('sm__inst_executed.avg.per_cycle_active') or 0:.2f} | "
                  f"{rec['report']} |")
    (ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    (ROOT / "profiles" / f"{tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[2:], sys.argv[1])
