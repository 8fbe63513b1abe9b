"""The NCCL collectives of the multi-GPU path, executed on the B200 box.

Only single-GPU boxes are available, so this runs a world-1 NCCL process
group (in a subprocess, so the pytest process keeps no process group) and
drives the exact collectives `parallel.py` issues at world > 1 -- the
all-gather of the layer-major pool arena (`_all_gather_rows` /
`gather_arena`, uint8 rows) and the MAX all-reduce of the per-layer key
maxima (`all_reduce_layer_max`, int32 bit patterns) -- on real pool tensors,
then checks the gathered pool decodes bit-identically. The world-2 logic
(sharding plan, padding, compaction, fault propagation) is covered by the
gloo tests in tests/test_parallel_cpu.py.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = textwrap.dedent(
    """
    import os, sys, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["PKV_ROOT"])
    import paper_2604_24971_b200 as pk
    from paper_2604_24971_b200 import parallel
    from paper_2604_24971_b200.pool import _Arena, _encode_layers

    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    assert dist.get_backend() == "nccl"
    dev = torch.device("cuda", 0)
    g = pk.ModelGeometry(num_layers=5, kv_heads=4, head_dim=128, seq_len=96)
    dump = pk.synth_gaussian_dump(g, seed=4, device=dev)
    ref = pk.build_pool(dump)

    # the arena all-gather, as issued at world > 1 (all_gather_into_tensor on uint8 rows)
    arena = _Arena(g, g.num_layers, "tensor", dev)
    _encode_layers([k for k, _ in dump.layers], [v for _, v in dump.layers], g, pk.GAUSSIAN_3BIT, None,
                   "tensor", device=dev, arena=arena)
    out = torch.empty_like(arena.flat)
    dist.all_gather_into_tensor(out, arena.flat)
    torch.cuda.synchronize()
    assert torch.equal(out, arena.flat)
    arena.flat.copy_(out)  # the gathered bytes, seen through the arena's field views
    n = g.elements_per_tensor
    for i in range(g.num_layers):
        assert torch.equal(arena.k_codes[i][:n], ref.layer_blocks(i)[0].codes.reshape(-1))
        assert torch.equal(arena.v_packed[i][:ref.layer_blocks(i)[1].packed.numel()], ref.layer_blocks(i)[1].packed)

    # the per-layer key-max all-reduce (int32 bit patterns, MAX)
    mx = parallel.local_key_max([k for k, _ in dump.layers], dev)
    red = mx.clone()
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    torch.cuda.synchronize()
    assert torch.equal(red, mx)
    # head-sharded build with the reduced maxima == the whole pool
    hp = parallel.build_pool_head_sharded(dump)
    for i in range(g.num_layers):
        assert hp.layer_blocks(i)[0].scale == ref.layer_blocks(i)[0].scale
        assert torch.equal(hp.layer_blocks(i)[0].codes, ref.layer_blocks(i)[0].codes)
    # decoded views of the layer-sharded pool equal the whole pool's
    sp = parallel.build_pool_sharded(dump)
    a, b = ref.attach(16), sp.attach(16)
    for i in range(g.num_layers):
        (ka, va), (kb, vb) = a.get_kv_for_layer(i), b.get_kv_for_layer(i)
        assert torch.equal(ka.values, kb.values) and torch.equal(va.values, vb.values)
    dist.destroy_process_group()
    print("NCCL-OK", torch.cuda.nccl.version())
    """
)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_collectives_of_the_sharded_pool():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0", PKV_ROOT=str(ROOT))
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "NCCL-OK" in r.stdout
