make -s all > /dev/null 2>&1 || exit 1
FMM2D_TREE_TRACE=1 timeout 600 python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, workloads as W
from paper_1006_2269_b200 import Fmm2d
c=W.CONFIGS["C5"]; z_np,_=W.make_config("C5"); z=torch.from_numpy(z_np).cuda()
for i in range(3):
    p=Fmm2d(z, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=True)
    s=p.stats(); print("tree", s["t_tree_ms"], "lists", s["t_lists_ms"], flush=True); p.close()
PY
