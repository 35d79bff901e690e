"""Summaries of ncu outputs for profiles/ (run in the build container).

    python scripts/summarize_ncu.py launches gpurun_out/launches_c2.csv > profiles/rNN_launches_summary.txt
    python scripts/summarize_ncu.py full gpurun_out/tc3_full.ncu-rep > profiles/rNN_tc3_full.txt
"""
import collections
import csv
import io
import subprocess
import sys


def to_ms(v, unit):
    v = float(v.replace(",", ""))
    return {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6) * v


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = to_ms(d["Metric Value"], d["Metric Unit"])
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
        total += ms
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)")
    print(f"# source: {path}; total {total:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    print(f"{'ms':>10} {'share':>6} {'count':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.3f} {100 * v[1] / total:5.1f}% {v[0]:6d}  {k}")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full --clock-control none, source: {path}")
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print(f"## {d.get('Kernel Name', '')[:140]}")
        for k in KEYS:
            if k in d:
                print(f"{k:80s} {d[k]:>16s} {units[hdr.index(k)]}")
        stalls = [(h, vals[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled") and h.endswith("ratio")]
        if stalls:
            print("# warp stall reasons (issue-stalled cycles per instruction)")
            for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:8]:
                print(f"  {h:78s} {v}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
