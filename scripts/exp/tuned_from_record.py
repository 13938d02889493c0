"""Write paper_2006_03031_b200/tuned/bert_dense_schedules.json from a tune_symbolic.py record."""
import json, sys
rec = json.load(open(sys.argv[1]))
out = {"source": "scripts/tune_symbolic.py on one B200 (full record: " + sys.argv[2] + ")",
       "procedure": rec["procedure"],
       "note": "tile_t = 0: the default DISPATCH.md rule won (no schedule registered)",
       "schedules": [{"op": s["op"], "N": s["N"], "K": s["K"], "tile_t": s["tile_t"], "split_max": s["split_max"],
                      "heldout_geomean_speedup_vs_default": s["heldout_geomean_speedup_vs_default"]}
                     for s in rec["schedules"]]}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out["schedules"]))
