"""Convert a per-rank pass timeline (scripts/timeline_mp.py output: per rank
{"ms", "passes": [[rank, kind, k, i, start ms, end ms], ...]}) into the
reference's Gantt JSON and its metric definitions (plan.gantt_measured_text /
plan.metrics_measured), checking the pass ids against the schedule.
usage: timeline_to_gantt.py TIMELINE.json P M N [V]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14519_b200 import plan as P  # noqa: E402

path, p, m, n = sys.argv[1], *map(int, sys.argv[2:5])
v = int(sys.argv[5]) if len(sys.argv) > 5 else 1
ranks = json.load(open(path))
sched = P.gen_slimpipe(p, v, m, n)
ids = {(q["kind"], q["microbatch"], q["slice"], q["device"]): q["id"] for q in sched["passes"]}
rows = []
for d, r in enumerate(ranks):
    out = []
    for rank, kind, k, i, s, e in r["passes"]:
        assert rank == d
        out.append((ids[(kind, k, i, d + 1)], s, e))
    rows.append(out)
stem = path[:-5] if path.endswith(".json") else path
Path(stem + ".gantt.json").write_text(P.gantt_measured_text(p, v, m, n, rows))
Path(stem + ".metrics.json").write_text(json.dumps(P.metrics_measured(p, v, m, n, rows), indent=1) + "\n")
print("wrote", stem + ".gantt.json", stem + ".metrics.json")
