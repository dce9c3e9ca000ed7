python tools/seg_build_c5.py c5
python -X importtime -c "pass" 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/seg_c5.csv python tools/seg_build_c5.py c5 > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/seg_c5.csv 1 | tail -40
python - <<'PY'
import cProfile, pstats, sys, io
sys.argv=['x','c5']
sys.path.insert(0,'.')
import torch
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import SegLayout
A = synth.laplacian5(2828); n=A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
B = P.permute_csr(A, p_r, p_c)
SegLayout(B, 2); torch.cuda.synchronize()
pr=cProfile.Profile(); pr.enable(); SegLayout(B, 2); torch.cuda.synchronize(); pr.disable()
s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats('cumulative').print_stats(25); print(s.getvalue()[:4000])
PY
