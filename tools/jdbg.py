import sys, numpy as np
sys.path.insert(0, '.')
from paper_1708_04174_b200 import SosAdmm
from sosgen import make_config
prob = make_config("pop6")
g = SosAdmm.from_problem(prob)
g.iterate(3)
g.iterate(200)
