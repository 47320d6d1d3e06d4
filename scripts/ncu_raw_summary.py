"""Markdown table of key metrics from `ncu -i rep --page raw --csv` exports (one per kernel)."""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "lts__t_requests_srcunit_tex_op_red.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"\n### {path.split('/')[-1].replace('.raw.csv', '')}: {d.get('Kernel Name', '')[:90]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in WANT:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        st = sorted(((float(d[k]), k) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled")
                     and not k.endswith("not_issued") and d[k] not in ("", "n/a")), reverse=True)[:5]
        print("| top stall reasons (pc samples) | " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {int(v)}" for v, k in st) + " | |")
