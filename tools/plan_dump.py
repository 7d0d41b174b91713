"""Print a plan's launches (BCSS_PLAN_DUMP) without running it: python tools/plan_dump.py m n p ba bc"""
import os
import sys

sys.path.insert(0, ".")
os.environ["BCSS_PLAN_DUMP"] = "1"
import paper_1301_7744_b200 as bs

m, n, p, ba, bc = (int(v) for v in sys.argv[1:6])
plan = bs.SttsmPlan(m, n, p, ba, bc)
print(plan.stats())
