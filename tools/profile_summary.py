"""Write the judged profile summaries for a round from a gpurun_out/<tag> directory:
profiles/<round>_ncu_summary.txt   key ncu --set full metrics + stall mix per profiled kernel
profiles/<round>_launch_shares.txt kernel share of the launch list (ncu gpu__time_duration pass)
profiles/<round>_launches.csv      the launch list itself
profiles/ncu_traffic.json          dram bytes per launch per kernel (read by bench.py)
profiles/<round>_bench.json        the bench line of that run
"""
import csv
import io
import json
import pathlib
import re
import shutil
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent


def short(name: str) -> str:
    m = re.search(r"::(\w+)(<[^>]*>)?\(", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main(src: str, rnd: str):
    src = pathlib.Path(src)
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    rep = src / "prof.ncu-rep"
    if rep.exists():
        txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                             capture_output=True, text=True).stdout
        (prof / f"{rnd}_ncu_summary.txt").write_text(
            f"# ncu --set full --clock-control none of tools/prof_kernels.py (gpurun_out/{src.name})\n" + txt)
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, data = rows[0], rows[2:]
        traffic = {}
        for r in data:
            k = short(r[hdr.index("Kernel Name")]).split("<")[0]
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            unit = rows[1][hdr.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            traffic.setdefault(k, []).append((rd + wr) * scale)
        tj = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches_profiled": len(v), "source": f"{rnd} ncu"}
              for k, v in traffic.items()}
        old = json.loads((prof / "ncu_traffic.json").read_text()) if (prof / "ncu_traffic.json").exists() else {}
        old.update(tj)
        (prof / "ncu_traffic.json").write_text(json.dumps(old, indent=1) + "\n")
    lc = src / "launches.csv"
    if lc.exists():
        shutil.copy(lc, prof / f"{rnd}_launches.csv")
        lines = [ln for ln in lc.read_text().splitlines() if ln.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr, data = rows[0], rows[1:]
        tot, per = 0.0, {}
        for r in data:
            if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            v = float(r[hdr.index("Metric Value")].replace(",", ""))
            k = short(r[hdr.index("Kernel Name")])
            per.setdefault(k, [0, 0.0])
            per[k][0] += 1
            per[k][1] += v
            tot += v
        out = [f"# kernel shares of the ncu launch list (gpu__time_duration.sum, cold-cache, serialised) — {src.name}",
               f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}"]
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            out.append(f"{k:60s} {n:8d} {t / 1e6:10.3f} {100 * t / tot:6.1f}% {t / n / 1e3:9.1f}")
        (prof / f"{rnd}_launch_shares.txt").write_text("\n".join(out) + "\n")
    bj = src / "bench.json"
    if bj.exists() and bj.read_text().strip():
        shutil.copy(bj, prof / f"{rnd}_bench.json")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
