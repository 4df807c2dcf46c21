import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2309_04841_b200 import QaoaSimulator, hamming_weight_state
from paper_2309_04841_b200.problems import portfolio_terms
n=14
sim = QaoaSimulator(terms=portfolio_terms(n), mixer="xy-ring")
res = sim.simulate_qaoa([0.3],[0.2], initial=hamming_weight_state(n, 7))
print(sim.get_expectation(res))
