cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-sf}; mkdir -p $o
cat > /tmp/sfrun.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, dgm_inputs as di
from paper_1104_4208_b200 import Context
from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE
p = int(sys.argv[1])
m = di.kuhn_mesh(12, periodic=(True, True, True), jitter=0.1, seed=1)
cm, en = di.curved_mesh(m, 0.03)
c = Context(cm.xyz, cm.tet, p, rep=m.rep, edge_nodes=en)
E = c.to_device(di.random_coefficients(m.n_tet, p, 1)); H = c.to_device(di.random_coefficients(m.n_tet, p, 2))
c.dgm_step(E, H, 1e-4, 1)
for _ in range(3): c.dgm_step_ex(E, H, 1e-4, 1, DGM_STEP_CONTINUE)
torch.cuda.synchronize()
PY
for p in 6 10; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $o/launches_curved_p$p.csv python /tmp/sfrun.py $p > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sumfact -s 2 -c 1 -o $o/sumfact_p10 python /tmp/sfrun.py 10 > $o/ncu_full.log 2>&1; tail -1 $o/ncu_full.log
