"""Summarise ncu launch lists (gpu__time_duration + dram bytes per launch) into
profiles/traffic.json and a per-kernel text table.

    python tools/make_traffic.py gpurun_out/r01b profiles/r01_launches.txt

traffic.json maps workload -> library kernel kind -> mean DRAM bytes per launch
(read + write), the `roofline.traffic` bench.py reports.  ncu replays every
launch cold and serialised, so its durations are for the kernel's SHARE of the
step, not absolute timings."""
import csv
import json
import os
import re
import sys
from collections import OrderedDict, defaultdict

KIND = [(r"rec_fwd_kernel", "rec_fwd"), (r"rec_bwd_kernel", "rec_bwd"), (r"lti2?_prep_kernel", "lti_prep"),
        (r"state_carry_kernel", "state_carry"), (r"tv_fir_|tv_add_kernel", "tv_fir"), (r"lti2?_fwd_kernel", "lti_fwd"),
        (r"lti2?_bwd", "lti_bwd"),
        (r"tv_phi2?_kernel", "tv_phi"), (r"tv_(group|groupchain|expand|chain)_kernel", "tv_chain"),
        (r"tv_seq_kernel<[^,]+, *(\(int\))?\d+, *(\(int\))?0>", "tv_fwd"),
        (r"tv_seq_kernel<[^,]+, *(\(int\))?\d+, *(\(int\))?1>", "tv_bwd_agg"),
        (r"tv_seq_kernel<[^,]+, *(\(int\))?\d+, *(\(int\))?2>", "tv_bwd"),
        (r"tv_seq_kernel<[^,]+, *(\(int\))?\d+, *(\(int\))?3>", "tv_wagg"),  # TV_FWD_AGG: fp64 w re-run
        (r"(skew_kernel|unskew_kernel|zi_add_kernel|zf_kernel|gy_eff_kernel|tail_kernel)", "tv_skew"),
        (r"dg_prep_kernel", "diag_prep"), (r"dg_agg_kernel", "diag_agg"), (r"dg_scan_kernel", "diag_scan"),
        (r"dg_fwd_emit_kernel", "diag_fwd"), (r"dg_bwd_emit_kernel", "diag_bwd"), (r"dg_reduce_kernel", "diag_red")]


def kind_of(name):
    for pat, k in KIND:
        if re.search(pat, name):
            return k
    return None


def parse(path):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[i:]))
    hdr = rows[0]
    per = OrderedDict()
    for r in rows[1:]:
        x = dict(zip(hdr, r))
        key = (x["ID"], x["Kernel Name"])
        v = float(x["Metric Value"].replace(",", ""))
        unit = x["Metric Unit"]
        if unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        elif unit == "Kbyte":
            v *= 1e3
        elif unit == "Mbyte":
            v *= 1e6
        elif unit == "Gbyte":
            v *= 1e9
        per.setdefault(key, {})[x["Metric Name"]] = v
    return per


def main():
    src, out_txt = sys.argv[1], sys.argv[2]
    traffic, lines = {}, []
    for f in sorted(os.listdir(src)):
        m = re.match(r"launches_(\w+)\.csv$", f)
        if not m:
            continue
        w = m.group(1)
        agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
        for (_, name), d in parse(os.path.join(src, f)).items():
            k = kind_of(name)
            if k is None:
                continue
            a = agg[k]
            a[0] += 1
            a[1] += d.get("gpu__time_duration.sum", 0.0)
            a[2] += d.get("dram__bytes_read.sum", 0.0)
            a[3] += d.get("dram__bytes_write.sum", 0.0)
        traffic[w] = {k: (a[2] + a[3]) / a[0] for k, a in agg.items()}
        fk = next(k for k in ("tv_fwd", "rec_fwd", "lti_fwd", "diag_fwd") if k in agg)
        steps = agg[fk][0]
        tot = sum(a[1] for a in agg.values()) / steps
        lines.append(f"== {w}: {steps} steps, ncu cold-cache serialised replay; per launch and share of the step")
        for k, a in agg.items():
            n = a[0]
            lines.append(f"   {k:11s} launches/step {n / steps:4.1f}  {a[1] / n / 1e3:9.2f} us/launch  "
                         f"share {a[1] / steps / tot:6.1%}  dram read {a[2] / n / 1e6:9.2f} MB  "
                         f"write {a[3] / n / 1e6:9.2f} MB per launch")
    os.makedirs("profiles", exist_ok=True)
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
