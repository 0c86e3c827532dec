"""Development aid: which reference-timeout sites of a workload the engine
decides within the per-query budget (one query at a time), and batch parity
of the rest."""
import sys, time, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries, mismatches, timed_out
from paper_2603_24595_b200.engine import SiteChecker
name = sys.argv[1]
doc = load(name); qs = queries(doc)
chk = SiteChecker(device=0)
hard = [i for i, s in enumerate(doc["sites"]) if timed_out(s)]
for i in hard:
    t = time.time(); r = chk.check(*qs[i])
    print(i, doc["sites"][i]["site"], doc["sites"][i]["line"], r.status, doc["sites"][i]["z3_verdict"], "%.1fs" % (time.time() - t), flush=True)
rest = [i for i in range(len(qs)) if i not in hard]
t = time.time()
res = chk.check_queries([qs[i] for i in rest])
sub = dict(doc); sub["sites"] = [doc["sites"][i] for i in rest]
print("rest", len(rest), "mismatches", mismatches(sub, res), "%.2fs" % (time.time() - t))
chk.close()
