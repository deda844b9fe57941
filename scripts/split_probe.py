"""Within-step pipelining probe: one bench step (K2 for all slots, then K3
and K1 over `parts` slot blocks) with block b's K1 on stream B overlapping
block b+1's K3 on stream A.  L2 flushed between steps, CUDA events around
each step; prints ms per step for parts = 1, 2, 4."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import L2_FLUSH_BYTES, SLOTS, make_cell_agent, synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CodebookEngine, DevicePolicy, _native  # noqa: E402

cell, agent = make_cell_agent()
allocs, eps = synthetic_inputs(cell, SLOTS)
pol = DevicePolicy(agent.actor, "fp32")
eng = CodebookEngine(pol, cell, max_slots=SLOTS, with_tree=True)
al, ep = torch.from_numpy(allocs).cuda(), torch.from_numpy(eps).cuda()
lib = _native.lib()
cap, e = cell.num_branches, cell.num_embb
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
raw, books, nodes = eng.raw, eng.codebooks, eng.node_state


def step(parts):
    _native.check(lib.cyr_actor_forward_device(pol.handle, al.data_ptr(), SLOTS, cell.total_scs,
                                               cap, raw.data_ptr(), sa.cuda_stream))
    per = SLOTS // parts
    for b in range(parts):
        s0 = b * per
        _native.check(lib.cyr_codebook_from_raw_device(
            pol.handle, raw[s0 * cap:].data_ptr(), al[s0:].data_ptr(), ep[s0:].data_ptr(), per,
            cell.total_scs, cell.urllc_sc_len, books[s0:].data_ptr(), None, None, None, None,
            eng.status.data_ptr(), sa.cuda_stream))
        ev = torch.cuda.Event()
        ev.record(sa)
        sb.wait_event(ev)
        _native.check(lib.cyr_tree_expand_device(books[s0:].data_ptr(), per, e, cap,
                                                 cell.minislots, nodes[s0:].data_ptr(),
                                                 sb.cuda_stream))
    done = torch.cuda.Event()
    done.record(sb)
    sa.wait_event(done)


for parts in (1, 2, 4, 1, 2, 4):
    for _ in range(3):
        step(parts)
    torch.cuda.synchronize()
    times = []
    for i in range(10):
        with torch.cuda.stream(sa):
            flush.fill_(i)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(sa)
        step(parts)
        t1.record(sa)
        torch.cuda.synchronize()
        times.append(t0.elapsed_time(t1))
    eng.check()
    print(f"parts={parts}: {np.mean(times) * 1e3:.1f} us per step")
