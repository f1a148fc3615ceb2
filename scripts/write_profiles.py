"""Turn the gpurun_out/ captures of scripts/gpu_profiles.sh into profiles/
summaries (committed) and profiles/<tag>_traffic.json (read by bench.py)."""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import ncu_summary as S

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = os.path.join(ROOT, "gpurun_out")
prof = os.path.join(ROOT, "profiles")
lc = os.path.join(out, f"{tag}_launches.csv")
if os.path.exists(lc):
    open(os.path.join(prof, f"{tag}_launches.txt"), "w").write(S.launches(lc) + "\n")
traffic = {"source": "ncu --set full --clock-control none, one launch each; bench.py config 2 (K=100k, 1024 rx, 90x360); "
                     "k_cov_signal from the config-3 leg (K=500k)"}
for name in ("train", "train_l1", "joint"):  # scripts/gpu_profiles_train.sh
    lc = os.path.join(out, f"{tag}_{name}_launches.csv")
    if os.path.exists(lc):
        open(os.path.join(prof, f"{tag}_{name}_launches.txt"), "w").write(S.launches(lc) + "\n")


def source_hotspots(rep, rows_per_launch=None, top=30):
    """Per CUDA source line: warp instructions and stall-sample share (ncu source page, -lineinfo)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    recs, fname = [], "?"
    for r in csv.reader(txt.splitlines()):
        if r and r[0] == "File Name":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0].isdigit():
            try:
                recs.append((fname, int(r[0]), r[1].strip()[:88], int(r[4]), int(r[7])))
            except ValueError:
                pass
    tot_s = sum(x[3] for x in recs) or 1
    tot_i = sum(x[4] for x in recs) or 1
    lines = [f"source-level hotspots of {os.path.basename(rep)} (ncu source page; instructions and stall samples "
             f"attributed to CUDA lines via -lineinfo)",
             f"attributed warp instructions: {tot_i}, stall samples: {tot_s}",
             "   line  instr%  stall%  source"]
    for x in sorted(recs, key=lambda x: -x[3])[:top]:
        lines.append(f"  {x[1]:5d}  {100 * x[4] / tot_i:5.1f}  {100 * x[3] / tot_s:5.1f}   {x[2]}")
    return "\n".join(lines) + "\n"


rep = os.path.join(out, f"{tag}_k_cond_tc.ncu-rep")
if os.path.exists(rep):
    open(os.path.join(prof, f"{tag}_k_cond_tc_source.txt"), "w").write(source_hotspots(rep))

for k in ["k_cond_tc", "k_fle_gemm", "k_composite_tc", "k_walk", "k_tx_prep", "k_cov_signal", "k_tile_scatter",
          "k_emit_entries", "k_radix_scatter", "k_cond_bwd_rows", "k_cond_bwd_grads", "k_cond_bwd_tc",
          "k_cond_grads_tc", "k_composite_T", "k_bwd_walk"]:
    rep = os.path.join(out, f"{tag}_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    open(os.path.join(prof, f"{tag}_{k}.txt"), "w").write(S.report(rep) + "\n")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
             "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}

    def get(m):  # value in base units (bytes, microseconds)
        if m not in h:
            return None
        i = h.index(m)
        return float(v[i].replace(",", "")) * scale.get(u[i], 1.0)

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    dur = get("gpu__time_duration.sum")
    traffic[k] = {"dram_bytes_per_launch": (rd + wr) if rd is not None else None,
                  "duration_us": dur,
                  # pipe evidence of the same launch (percent of peak sustained, active cycles)
                  "dram_gbps": (rd + wr) / (dur * 1e3) if rd is not None and dur else None,
                  "fp32_pipe_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                  "fp32_inst_pct": get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                  "tensor_pipe_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  "fp64_pipe_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                  "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
json.dump(traffic, open(os.path.join(prof, f"{tag}_traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
