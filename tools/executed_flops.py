"""FP64 flops the step kernels execute per solve, from an ncu metric list over
every step-kernel launch of one solve (report the executed rate
beside the method's algorithmic model).

  ncu --metrics <METRICS> --clock-control none -k regex:step_kernel --csv \
      --log-file launches.csv python tools/profile_step.py cfg4
  python tools/executed_flops.py cfg4 launches.csv [profiles/executed_flops.json]

flop = 2 * DFMA + DMUL + DADD thread instructions (predicated-on) + 512 per
DMMA m8n8k4 warp instruction (8 x 8 x 4 multiply-adds). Merges the result
for the workload into the JSON file bench.py reads.
"""
import collections
import csv
import json
import os
import sys

METRICS = ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
DMMA = os.environ.get("DMMA_METRIC", "smsp__inst_executed_pipe_fp64_op_dmma.sum")


def main():
    name, path = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "executed_flops.json")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iid, im, iv = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
    tot = collections.Counter()
    for d in per.values():
        for k, v in d.items():
            tot[k] += v
    flop = 2 * tot[METRICS[0]] + tot[METRICS[1]] + tot[METRICS[2]] + 512 * tot.get(DMMA, 0.0)
    rec = {"flop_per_solve": flop, "launches": len(per), "dfma": tot[METRICS[0]], "dmul": tot[METRICS[1]],
           "dadd": tot[METRICS[2]], "dmma_warp_inst": tot.get(DMMA), "dmma_metric": DMMA,
           "source": "ncu --metrics (thread-level FP64 SASS counts + DMMA) over all %d step-kernel launches of one "
                     "%s solve (tools/executed_flops.py)" % (len(per), name)}
    allj = json.load(open(out)) if os.path.exists(out) else {}
    allj[name] = rec
    json.dump(allj, open(out, "w"), indent=1)
    print(json.dumps({name: rec}))


if __name__ == "__main__":
    main()
