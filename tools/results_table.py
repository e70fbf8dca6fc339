"""Markdown results table from bench JSON lines (one file per workload).

    python tools/results_table.py DIR [c5 c4 ...]   -> prints the table used in DESIGN.md section 7
"""
import glob
import json
import os
import sys

ORDER = ["c5", "c4", "c2", "c1", "c3", "f1", "f2", "f2t", "f3"]


def load(path):
    for line in reversed(open(path).read().strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def traffic_table():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def main():
    d = sys.argv[1]
    tt = traffic_table()
    names = sys.argv[2:] or ORDER
    rows = ["| Workload | µs / step | samples/s | dominant kernel | its achieved GB/s (algorithmic) | roofline frac | "
            "DRAM bytes / launch (ncu) | e2e samples/s | oracle samples/s (cores) |",
            "|---|---|---|---|---|---|---|---|---|"]
    for w in names:
        fs = glob.glob(os.path.join(d, f"bench_{w}.json")) + glob.glob(os.path.join(d, f"b_{w}.json"))
        if not fs:
            continue
        j = load(fs[0])
        if j is None:
            continue
        r = j["roofline"]
        cb = j.get("cpu_baseline") or {}
        e2e = (j.get("e2e") or {}).get("value")
        tr = tt.get(w, {}).get(r.get("kernel")) or r.get("traffic")
        rows.append(f"| {w} ({j['config'].get('workload', '')[:40]}) | {j['ms_per_step'] * 1e3:.1f} | {j['value']:.3g} | "
                    f"`{r.get('kernel')}` | {r['achieved']:.0f} | {r['frac']:.3f} | "
                    f"{'%.3g' % tr if tr else 'n/a'} | {e2e:.3g} | "
                    f"{cb.get('value', float('nan')):.3g} ({cb.get('cores', '?')}) |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
