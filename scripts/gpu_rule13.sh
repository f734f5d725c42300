cd $GRAFT_REPO_ROOT
for n in 24 31; do
timeout 120 python tools/probe_qft3.py $n 2>&1 | tail -1
QSIM_FORCE_QFT13=1 timeout 120 python tools/probe_qft3.py $n 2>&1 | tail -1
done
for m in 16; do
python - <<'PY'
import sys, os, json
sys.path.insert(0, '.')
from paper_quant_ph_0201042_b200 import qsim as Q
for m in (12, 16, 20, 24):
    h = Q.qsim_create(28); Q.qsim_init_gaussian(h, 3)
    for _ in range(2): Q.qsim_qft(h, 0, m, False)
    Q.qsim_sync(h); Q.qsim_profile(h, True)
    for _ in range(3): Q.qsim_qft(h, 0, m, False)
    p = Q.qsim_profile_json(h); l = p.pop('_launches')
    print(json.dumps({"n": 28, "m": m, "force13": os.environ.get("QSIM_FORCE_QFT13"), "ms": round(sum(x[1] for x in l) / 3, 4), "kernels": sorted(set(x[0] for x in l))}))
    Q.qsim_destroy(h)
PY
done
QSIM_FORCE_QFT13=1 python - <<'PY'
import sys, os, json
sys.path.insert(0, '.')
from paper_quant_ph_0201042_b200 import qsim as Q
for m in (12, 16, 20, 24):
    h = Q.qsim_create(28); Q.qsim_init_gaussian(h, 3)
    for _ in range(2): Q.qsim_qft(h, 0, m, False)
    Q.qsim_sync(h); Q.qsim_profile(h, True)
    for _ in range(3): Q.qsim_qft(h, 0, m, False)
    p = Q.qsim_profile_json(h); l = p.pop('_launches')
    print(json.dumps({"n": 28, "m": m, "force13": os.environ.get("QSIM_FORCE_QFT13"), "ms": round(sum(x[1] for x in l) / 3, 4), "kernels": sorted(set(x[0] for x in l))}))
    Q.qsim_destroy(h)
PY
