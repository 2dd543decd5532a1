"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections, csv, sys

UNIT_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short_name(full):
    s = full.split("(")[0].replace("void ", "").strip()
    depth, parts, cur = 0, [], ""
    for ch in s:  # split on '::' at template depth 0
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        if depth == 0 and cur.endswith(":") and ch == ":":
            parts.append(cur[:-1])
            cur = ""
            continue
        cur += ch
    parts.append(cur)
    last = parts[-1]
    if "<" in last and len(last) > 60:
        last = last.split("<")[0] + "<...>"
    return last


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    return [(short_name(r[ki]), float(r[vi].replace(",", "")) * UNIT_US.get(r[ui], 1.0))
            for r in rows[1:] if len(r) > vi]


if __name__ == "__main__":
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in rows:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {c:8d} {t:10.1f} {t / c:9.2f} {t / tot:6.3f}")
