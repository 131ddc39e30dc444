"""Copy one gpu_check.sh run into profiles/ under a tag (bench line, reference
arm, launch list, ncu details, per-phase summaries) and refresh
profiles/ncu_traffic.json (the bench's roofline.traffic source).

    python tools/save_profiles.py gpurun_out/<dir> <tag> [round prefix, default r02]
"""
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as ns  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNEL_SRC = os.path.join(ROOT, "paper_2605_07238_b200", "csrc", "fate_score_v6.cuh")


def main(src, tag, rnd="r02"):
    prof = os.path.join(ROOT, "profiles")
    for name, dst in (("bench.json", "bench.json"), ("bench_ref.json", "reference_arm.json"),
                      ("launches_c5.csv", "launches_c5.csv")):
        if os.path.exists(os.path.join(src, name)):
            shutil.copy(os.path.join(src, name), os.path.join(prof, f"{rnd}_{tag}_{dst}"))
    traffic = {"_comment": f"dram__bytes_read.sum + dram__bytes_write.sum of one fate_score "
                           f"launch (ncu --set full); kernel {tag} (profiles/{rnd}_{tag}_*)"}
    items = {"c5": 102400, "c4": 80000}
    for k, key in (("c5", "c5_frontier"), ("c4", "c4_sweep")):
        rep = os.path.join(src, f"{k}_full.ncu-rep")
        if not os.path.exists(rep):
            continue
        with open(os.path.join(prof, f"{rnd}_{tag}_{k}_details.csv"), "w") as fh:
            subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], stdout=fh, check=True)
        with open(os.path.join(prof, f"{rnd}_{tag}_{k}_summary.txt"), "w") as fh:
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep,
                            KERNEL_SRC, str(items[k])], stdout=fh, check=True)
        m = ns.raw_metrics(rep)
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        tot = sum(float(m[x][0]) * mult[m[x][1]] for x in ("dram__bytes_read.sum",
                                                            "dram__bytes_write.sum"))
        traffic[key] = int(round(tot))
    with open(os.path.join(prof, "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=2)
    print(json.dumps(traffic))
    # warp instructions per launch (issue-rate ceiling of the bench's roofline)
    inst = {"_comment": f"smsp__inst_executed.sum (warp instructions) of one fate_score launch; "
                        f"kernel {tag}"}
    for k, key in (("c5", "c5_frontier"), ("c4", "c4_sweep")):
        rep = os.path.join(src, f"{k}_full.ncu-rep")
        if os.path.exists(rep):
            inst[key] = int(float(ns.raw_metrics(rep)["smsp__inst_executed.sum"][0]))
    with open(os.path.join(prof, "ncu_instructions.json"), "w") as fh:
        json.dump(inst, fh, indent=2)
    print(json.dumps(inst))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(sys.argv[3:4]))
