"""Key metrics of an `ncu --set full` capture, as text for profiles/.

usage: python tools/ncu_summary.py <file.ncu-rep> [title]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst executed"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst executed"),
    ("sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA pipe active"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor (tc) pipe active"),
    ("lts__t_bytes.sum.per_second", "L2 throughput"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA (fp32/int) pipe active"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math throttle / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not selected / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall MIO throttle / issue"),
]


def to_json(rows, head, commit, capture):
    """profiles/fit3_profile.json for bench.py: the first k_fit3 launch of the capture."""
    import json

    for r in rows[2:]:
        d = dict(zip(head, r))
        if "k_fit3" not in d.get("Kernel Name", ""):
            continue
        num = lambda k: float(d[k].replace(",", "")) if k in d else None  # noqa: E731
        mb = 1e6  # ncu reports Mbyte here
        return {"kernel": d["Kernel Name"], "commit": commit, "capture": capture,
                "duration_ms": num("gpu__time_duration.sum"),
                "dram_bytes_per_launch": (num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) * mb,
                "fp64_pipe_active_frac": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100.0,
                "issue_active_frac": num("sm__issue_active.avg.pct_of_peak_sustained_elapsed") / 100.0}
    return None


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    if "--json" in sys.argv:
        import json

        commit = sys.argv[sys.argv.index("--json") + 1]
        print(json.dumps(to_json(rows, head, commit, rep), indent=1))
        return
    print(f"# {title}")
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for key, label in KEYS:
            if key in d:
                print(f"  {label:32s} {d[key]:>16s} {u.get(key, '')}")


if __name__ == "__main__":
    main()
