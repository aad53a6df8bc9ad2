"""Re-place a measured Gantt (bench.py --gantt) on one clock by first-pass
dependency: rank r's first pass starts where rank r-1's first pass ended
(bench.py now does this itself).  Used for the Gantts written by the bench
revision that shifted ranks by the GPUs' global timers (bench line key
"timeline_clock" with "causality_violation_ms"), which turned out to be
hundreds of ms apart across GPUs.  Rewrites <gantt> and <gantt>.metrics.json.

    python scripts/realign_gantt.py BENCH_LINE.json GANTT.json P M N SEQ_LEN
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14519_b200 import plan as P  # noqa: E402


def main():
    line_path, gantt_path = sys.argv[1], sys.argv[2]
    p, m, n, seq = (int(x) for x in sys.argv[3:7])
    line = json.loads(Path(line_path).read_text().strip().splitlines()[-1])
    shifted = (line.get("timeline_clock") or {}).get("offsets_ms") or [0.0] * p
    g = json.loads(Path(gantt_path).read_text())
    ids = {(q["kind"], q["microbatch"], q["slice"], q["stage"]): q["id"] for q in P.gen_slimpipe(p, 1, m, n)["passes"]}
    per_dev = []
    for r, row in enumerate(g["rows"]):
        spans = [(ids[(x["kind"], x["microbatch"], x["slice"], x["stage"])],
                  x["start"] - shifted[r], x["end"] - shifted[r]) for x in row]
        per_dev.append(spans)
    off = [0.0]
    for r in range(1, p):
        prev_end = min(per_dev[r - 1], key=lambda x: x[1])[2] + off[r - 1]
        off.append(prev_end - min(per_dev[r], key=lambda x: x[1])[1])
    per_dev = [[(i, s + off[r], e + off[r]) for i, s, e in spans] for r, spans in enumerate(per_dev)]
    Path(gantt_path).write_text(P.gantt_measured_text(p, 1, m, n, per_dev, False, seq))
    Path(gantt_path + ".metrics.json").write_text(json.dumps(P.metrics_measured(p, 1, m, n, per_dev, False, seq),
                                                             indent=1))
    print(gantt_path, "offsets", [round(o, 1) for o in off])


if __name__ == "__main__":
    main()
