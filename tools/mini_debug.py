import faulthandler, sys; faulthandler.enable()
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from common import problem
from paper_2511_00796_b200.engine import Engine
p=problem('c2_16gpu')
print('creating', flush=True)
e=Engine(p)
print('created', flush=True)
r=e.constrained_search([0,1,2,3], 3)
print(r, flush=True)
