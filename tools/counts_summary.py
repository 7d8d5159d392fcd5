"""profiles/traffic.json from the ncu counter CSVs of tools/profile_round.sh.

  python tools/counts_summary.py TAG [SRC_DIR]

Reads SRC_DIR/TAG_counts_{c3,c5,reset}.csv (default SRC_DIR gpurun_out), updates
the "c3:65536:1024", "c5:131072:1024" and "reset:c3:65536:1024" entries of
profiles/traffic.json (the counters bench.py reads for roofline.traffic and
roofline.components.fp64) and prints the markdown table rows of the counts summary.
"""
import csv
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
PARTICLE_STEPS = {"c3": 65536 * 25 * 1024, "c5": 131072 * 25 * 1024}
KEYS = {"c3": "c3:65536:1024", "c5": "c5:131072:1024", "reset": "reset:c3:65536:1024"}


def metrics(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, out = rows[0], {}
    i_name, i_val = hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        out[r[i_name]] = float(r[i_val].replace(",", ""))
    return out


def main():
    tag = sys.argv[1]
    src = pathlib.Path(sys.argv[2] if len(sys.argv) > 2 else ROOT / "gpurun_out")
    tj = ROOT / "profiles" / "traffic.json"
    traffic = json.loads(tj.read_text()) if tj.exists() else {}
    cap = (f"tools/profile_round.sh {tag}: ncu --metrics ... --clock-control none -k regex:step_kernel -s 3 -c 1 "
           "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-episode [--config c5]")
    for name in ("c3", "c5", "reset"):
        m = metrics(src / f"{tag}_counts_{name}.csv")
        fp64 = sum(m[f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum"] for k in ("dfma", "dmul", "dadd"))
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        if name == "reset":
            traffic[KEYS[name]] = dict(m, capture=f"tools/profile_round.sh {tag}: ncu --metrics ... -k regex:reset_kernel "
                                       "-c 1 (the ctor's reset of all 65,536 envs)")
            print(f"| reset_kernel (C3 ctor) | {m['gpu__time_duration.sum'] / 1e6:.2f} | "
                  f"{m['dram__bytes_read.sum'] / 1e9:.2f} + {m['dram__bytes_write.sum'] / 1e9:.2f} | — | — | — |")
            continue
        traffic[KEYS[name]] = {
            "dram_bytes_per_launch": dram, "fp64_thread_inst_per_launch": fp64,
            "dfma": m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"],
            "dmul": m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"],
            "dadd": m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"],
            "pipe_fp64_warp_inst": m["sm__inst_executed_pipe_fp64.sum"], "warp_inst": m["smsp__inst_executed.sum"],
            "thread_inst": m["smsp__thread_inst_executed.sum"], "ncu_duration_ns": m["gpu__time_duration.sum"],
            "fp64_source": f"ncu smsp__sass_thread_inst_executed_op_d{{fma,mul,add}}_pred_on.sum, one launch "
                           f"(profiles/{tag}_counts.md)",
            "capture": cap,
        }
        per = m["smsp__thread_inst_executed.sum"] / PARTICLE_STEPS[name]
        print(f"| step_kernel {name.upper()} | {m['gpu__time_duration.sum'] / 1e6:.2f} | "
              f"{m['dram__bytes_read.sum'] / 1e9:.2f} + {m['dram__bytes_write.sum'] / 1e9:.2f} = {dram / 1e9:.2f} | "
              f"{m['smsp__thread_inst_executed.sum'] / 1e9:,.1f} G | {per:.1f} | {fp64 / 1e9:.1f} G "
              f"({traffic[KEYS[name]]['dfma'] / 1e9:.1f} / {traffic[KEYS[name]]['dmul'] / 1e9:.1f} / "
              f"{traffic[KEYS[name]]['dadd'] / 1e9:.1f}) |")
    tj.write_text(json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    main()
