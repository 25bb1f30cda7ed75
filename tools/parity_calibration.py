"""Summarise a RQLP_PARITY_LOG file (tests/parity.py: one JSON record per graded factorisation)
into the calibration table of DESIGN.md §6:

  RQLP_PARITY_LOG=gpurun_out/parity_log.jsonl python -m pytest tests -m gpu -q
  python tools/parity_calibration.py gpurun_out/parity_log.jsonl profiles/r02_parity_calibration.json
"""
import json
import sys

recs = [json.loads(line) for line in open(sys.argv[1]) if line.strip()]
keys = ("L_abs_over_uL1", "L_rel_max", "Q_over", "P_over", "T_over", "QtQ", "PtP")
mx = {k: max((r[k] for r in recs if r.get(k) is not None), default=None) for k in keys}
arg = {k: next((r.get("tag") for r in recs if r.get(k) == mx[k]), None) for k in keys}
out = {"records": len(recs), "ties": sum(1 for r in recs if r.get("tie_step") is not None), "max": mx, "max_at": arg,
       "per_test": recs}
json.dump(out, open(sys.argv[2], "w"))
print(json.dumps({"records": out["records"], "ties": out["ties"], "max": mx, "max_at": arg}, indent=1))
