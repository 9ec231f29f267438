import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2305_12019_b200 import linalg as L
X = np.random.default_rng(0).standard_normal((2000, 20000))
for rep in range(2):
    G = L.gram(X, False)
print(G[0, 0])
