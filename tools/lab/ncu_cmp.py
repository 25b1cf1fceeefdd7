"""Side-by-side raw ncu metrics of the kernels in several reports.
usage: python tools/lab/ncu_cmp.py a.ncu-rep b.ncu-rep ... [-m substr,substr]"""
import csv, subprocess, sys, io
args = [a for a in sys.argv[1:] if not a.startswith("-m")]
pick = None
for a in sys.argv[1:]:
    if a.startswith("-m"):
        pick = a[2:].split(",")
KEYS = pick or ["gpu__time_duration.sum", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait"]
for rep in args:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:50]
        print("==", rep.split("/")[-1], name)
        for k in KEYS:
            for h, v in zip(hdr, r):
                if h == k:
                    print("   %-75s %s" % (k, v))
