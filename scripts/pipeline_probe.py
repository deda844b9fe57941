"""Cross-step pipelining probe: K2/K3 of step i+1 (stream A) overlapped with
K1 of step i (stream B), codebooks double-buffered.  Prints ms per step for
the serial and the pipelined schedule (CUDA events around K steps)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SLOTS, make_cell_agent, synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CodebookEngine, DevicePolicy, _native  # noqa: E402

cell, agent = make_cell_agent()
allocs, eps = synthetic_inputs(cell, SLOTS)
pol = DevicePolicy(agent.actor, "fp32")
eng = CodebookEngine(pol, cell, max_slots=SLOTS, with_tree=True)
al, ep = torch.from_numpy(allocs).cuda(), torch.from_numpy(eps).cuda()
lib = _native.lib()
cap, e = cell.num_branches, cell.num_embb
books = [torch.empty((SLOTS, cap + 1, e), dtype=torch.int32, device="cuda") for _ in range(2)]
raw = torch.empty((SLOTS * cap, 2 * e), dtype=torch.float32, device="cuda")
status = torch.zeros(4, dtype=torch.int32, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def k23(buf, st):
    _native.check(lib.cyr_actor_forward_device(pol.handle, al.data_ptr(), SLOTS, cell.total_scs, cap,
                                               raw.data_ptr(), st.cuda_stream))
    _native.check(lib.cyr_codebook_from_raw_device(pol.handle, raw.data_ptr(), al.data_ptr(),
                                                   ep.data_ptr(), SLOTS, cell.total_scs,
                                                   cell.urllc_sc_len, books[buf].data_ptr(), None,
                                                   None, None, None, status.data_ptr(),
                                                   st.cuda_stream))


def k1(buf, st):
    _native.check(lib.cyr_tree_expand_device(books[buf].data_ptr(), SLOTS, e, cap, cell.minislots,
                                             eng.node_state.data_ptr(), st.cuda_stream))


def serial(k):
    for i in range(k):
        k23(0, sa)
        k1(0, sa)


def pipelined(k):
    done23 = [torch.cuda.Event() for _ in range(2)]
    done1 = [torch.cuda.Event() for _ in range(2)]
    k23(0, sa)
    done23[0].record(sa)
    for i in range(k):
        if i + 1 < k:  # next step's codebooks first, into the other buffer
            nb = (i + 1) % 2
            if i >= 1:
                sa.wait_event(done1[nb])  # K1 of step i-1 has read that buffer
            k23(nb, sa)
            done23[nb].record(sa)
        sb.wait_event(done23[i % 2])
        k1(i % 2, sb)
        done1[i % 2].record(sb)
    sa.wait_stream(sb)


for name, fn in (("serial", serial), ("pipelined", pipelined)):
    fn(3)
    torch.cuda.synchronize()
    k = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(sa)
    fn(k)
    b.record(sa)
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / k:.3f} ms/step -> {SLOTS / (a.elapsed_time(b) / k) * 1e3:.0f} codebooks/s")
