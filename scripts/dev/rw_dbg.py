"""Dev tool: run LOD variants on a sequence of shapes in one process against the oracle."""
import sys, os
sys.path.insert(0, os.getcwd())
from tests.test_gpu_shapes import problems
import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from tests.helpers import rel_err
for arg in sys.argv[1:]:
    sh, vs = arg.split(":")
    shape = tuple(int(x) for x in sh.split(","))
    p, op = problems(shape, seed=1)
    for v in vs.split(","):
        try:
            rep = pb.march(p, pb.MarchConfig(dt=0.2, T=0.6, variant=v))
            orep = O.march(op, v, 0.2, 0.6)
            print(shape, v, "ok", rel_err(rep.final.data, orep.final), flush=True)
        except Exception as e:
            print(shape, v, "ERR", e, flush=True)
