"""Turn the ncu captures brought back in gpurun_out/ into the committed
summaries under profiles/ (run here, on the CPU box).

usage: python scripts/make_profiles.py <round tag> <dir written by scripts/profile_round.sh>
"""
import csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import ncu_summary as S  # noqa: E402

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_selected"]


def summarise(kind, path):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), kind, path],
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out)


def full_summary(rep, out_txt):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    lines = []
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        lines.append(f"kernel: {name}")
        for i, n in enumerate(h):
            if n in KEYS:
                lines.append(f"  {n:60s} {row[i]:>20s} {u[i]}")
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    return "\n".join(lines)


def main():
    """usage: make_profiles.py TAG DIR -- DIR holds the outputs of
    scripts/profile_round.sh (launches_cfg2.csv, traffic_<wl>.csv,
    full_<wl>.ncu-rep)."""
    tag, d = sys.argv[1], sys.argv[2]
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    L = summarise("launches", os.path.join(d, "launches_cfg2.csv"))
    with open(os.path.join(pdir, f"{tag}_launches_cfg2.json"), "w") as f:
        json.dump(L, f, indent=1)
    shutil.copy(os.path.join(d, "launches_cfg2.csv"), os.path.join(pdir, f"{tag}_launches_cfg2.csv"))
    for fn in sorted(os.listdir(d)):
        if fn.startswith("traffic_") and fn.endswith(".csv"):
            wl = fn[len("traffic_"):-4]
            T = summarise("traffic", os.path.join(d, fn))
            # the workload's dominant level kernel (k_level; k_pull for cfg3's bottom-up knows+)
            kname = max((n for n in T if n in ("k_level", "k_pull")), key=lambda n: T[n]["time_us"])
            k = T[kname]
            shards = " 64" if wl == "cfg5" else ""
            with open(os.path.join(pdir, f"traffic_{wl}.json"), "w") as f:
                json.dump({"kernel": kname, "dram_bytes_per_launch": k["dram_bytes_per_launch"],
                           "launches": k["launches"], "round": tag,
                           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                                     f"-k regex:'k_level|k_pull|k_count_total|k_clear_dense' over one COUNT "
                                     f"evaluation of each {wl} query "
                                     f"(scripts/prof_workload.py {wl}{shards}, RPQ_HOST_LOOP=1, PROF_NOSTATS=1)",
                           "all": T}, f, indent=1)
        if fn.startswith("full_") and fn.endswith(".ncu-rep"):
            wl = fn[len("full_"):-len(".ncu-rep")]
            print(full_summary(os.path.join(d, fn), os.path.join(pdir, f"{tag}_k_level_full_{wl}.txt")))
            shutil.copy(os.path.join(d, fn), os.path.join(pdir, f"{tag}_k_level_{wl}.ncu-rep"))


if __name__ == "__main__":
    main()
