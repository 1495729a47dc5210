#!/usr/bin/env python
"""Anatomy of one timed Kernelet step from `bench.py --trace-out` (device %globaltimer records
of every launch): how long each set of co-resident kinds ran, how long the critical kind (the
one with the largest solo work in the queue) was resident, how long no launch or only one launch
was resident, and the launch count.  CPU post-processing.

usage: python tools/step_anatomy.py TRACE.jsonl [OUT.json] [--critical MRIQ]"""
import collections
import json
import sys


def anatomy(recs, critical="MRIQ"):
    ev = []
    for r in recs:
        if not r.get("adm") or r["t1_us"] <= r["t0_us"]:
            continue
        ev.append((r["t0_us"], 1, r["kind"]))
        ev.append((r["t1_us"], -1, r["kind"]))
    ev.sort(key=lambda e: (e[0], e[1]))
    live = collections.Counter()
    by_set = collections.Counter()
    crit_us = idle_us = single_us = 0.0
    t_prev = ev[0][0] if ev else 0.0
    for t, d, k in ev:
        dt = t - t_prev
        if dt > 0:
            kinds = tuple(sorted(x for x, n in live.items() if n > 0))
            by_set[kinds] += dt
            if critical in kinds:
                crit_us += dt
            if not kinds:
                idle_us += dt
            if sum(live.values()) == 1:
                single_us += dt
        live[k] += d
        t_prev = t
    span = (ev[-1][0] - ev[0][0]) if ev else 0.0
    top = sorted(by_set.items(), key=lambda kv: -kv[1])[:25]
    return {"span_us": span, "launches": len(ev) // 2, "critical": critical, "critical_resident_us": crit_us,
            "critical_resident_frac": crit_us / span if span else 0.0, "idle_us": idle_us,
            "one_launch_resident_us": single_us,
            "by_resident_set_us": [{"kinds": list(k), "us": round(v, 1), "frac": round(v / span, 4)} for k, v in top]}


def main():
    argv = list(sys.argv[1:])
    crit = "MRIQ"
    if "--critical" in argv:
        i = argv.index("--critical")
        crit = argv[i + 1]
        del argv[i:i + 2]
    args = argv
    recs = [json.loads(line) for line in open(args[0]) if line.strip()]
    out = anatomy(recs, crit)
    s = json.dumps(out, indent=1)
    if len(args) > 1:
        open(args[1], "w").write(s)
    print(s)


if __name__ == "__main__":
    main()
