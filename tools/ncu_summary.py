"""Summarise an ncu --set full report: key throughput metrics + top stall sites."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def stalls(rep, n=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ia, isrc, iw = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
    tot = sum(float(r[iw] or 0) for r in data) or 1
    res = []
    for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:n]:
        br = sorted(((c, float(r[hdr.index(c)] or 0)) for c in cols), key=lambda kv: -kv[1])
        res.append((float(r[iw]) / tot * 100, r[ia][-5:], r[isrc][:70], br[0][0]))
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        m = raw(rep)
        for k in KEYS:
            if k in m:
                print(f"  {k:85s} {m[k][1]:>14s} {m[k][0]}")
        for pct, a, src, why in stalls(rep):
            print(f"  {pct:5.1f}% {a} {src:72s} {why}")
