"""Event timing of the Mode-T leaf scoring (cyr_tree_leaf_score_states_device)
on a cfg5-sized record array (823,543 leaves x 16 users)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_00167_b200 import CellConfig, tree  # noqa: E402

cell = CellConfig(780, 16, 130)
cap, m = cell.num_branches, cell.minislots
nodes = tree.num_nodes(cap, m)
states = torch.randint(0, 200, (1, nodes, 16), dtype=torch.int16, device="cuda")
al = torch.full((1, 16), 48, dtype=torch.int32, device="cuda")
margins = torch.full((1, 16), 0.3, dtype=torch.float64, device="cuda")
prob = torch.from_numpy(tree.admitted_count_probs(cell)).cuda()
for leaf_ok in (True, False):
    for _ in range(3):
        tree.score_leaf_states(states, cell, al, margins, prob, leaf_ok=leaf_ok)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        tree.score_leaf_states(states, cell, al, margins, prob, leaf_ok=leaf_ok)
    b.record()
    torch.cuda.synchronize()
    print(f"leaf_ok={leaf_ok}: {a.elapsed_time(b) / 20 * 1e3:.1f} us per call "
          f"({nodes} nodes, {(cap + 1) ** m} leaves)")
