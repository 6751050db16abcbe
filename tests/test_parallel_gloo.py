"""Keyframe-batch data parallelism on CPU with the gloo backend, world size 2.

Each rank computes per-view parameter gradients for its shard of a 4-keyframe batch (with the
CPU oracle standing in for the device kernels -- test-only injection), then runs the product
collective `parallel.allreduce_grads` (gradient rows summed, touched masks OR-ed through the
padding column of the same buffer) and applies one sparse Adam step.  The result must equal
the single-process batch oracle: sum of per-view gradients, union of touched, one
sparse_adam_step -- and both replicas must end bit-identical.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _scene():
    from paper_2507_04004_b200 import scenes
    return scenes.scene_room(2048, 64, 48, lidar=8, render_views=(0, 8, 16, 24))


def _view_grads(sc, rows, k):
    c = sc.cams[k]
    cam = O.Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"], c["trans_cw"])
    g = O.GaussianMap.from_rows(rows)
    out = O.forward(g, cam)
    _, gc, gd, go = O.mapping_loss(out.color, out.depth, out.opacity, sc.targets[k], sc.sparse_depths[k], 0.2, 0.005)
    grads, touched, _ = O.backward(g, out, gc, gd, go)
    return O.grads_to_rows(grads), touched


def _worker(rank, world, port, result_path, sparse=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_04004_b200 import parallel as PAR
    sc = _scene()
    rows = sc.rows.astype(np.float32).astype(np.float64)
    n = len(rows)
    acc = torch.zeros((n, 64), dtype=torch.float32)
    touched = torch.zeros(n, dtype=torch.uint8)
    for k in range(rank, 4, world):
        gr, t = _view_grads(sc, rows, k)
        acc[:, :59] += torch.as_tensor(gr, dtype=torch.float32)
        touched |= torch.as_tensor(t.astype(np.uint8))
    if sparse:
        PAR.allreduce_grads_sparse(acc, touched)
    else:
        PAR.allreduce_grads(acc, touched)
    st = O.AdamState()
    O.adam_rows(rows, acc[:, :59].double().numpy(), touched.numpy().astype(bool), st, O.default_lrs(3.0))
    np.save(result_path.format(rank), rows)
    np.save(result_path.format(f"t{rank}"), touched.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(600)
@pytest.mark.parametrize("sparse", [False, True])
def test_batch_dp_two_ranks_matches_batch_oracle(tmp_path, sparse):
    """Dense (one collective, flag in the padding column) and two-phase sparse allreduce."""
    path = str(tmp_path / "rows_{}.npy")
    mp.spawn(_worker, args=(2, _free_port(), path, sparse), nprocs=2, join=True)
    r0 = np.load(path.format(0))
    r1 = np.load(path.format(1))
    assert np.array_equal(r0, r1), "replicas diverged"
    # single-process batch oracle
    sc = _scene()
    rows = sc.rows.astype(np.float32).astype(np.float64)
    total = np.zeros((len(rows), 59))
    union = np.zeros(len(rows), bool)
    for k in range(4):
        gr, t = _view_grads(sc, rows, k)
        total += gr.astype(np.float32)
        union |= t
    assert np.array_equal(np.load(path.format("t0")).astype(bool), union)
    st = O.AdamState()
    O.adam_rows(rows, total.astype(np.float32).astype(np.float64), union, st, O.default_lrs(3.0))
    delta_dp = r0 - sc.rows.astype(np.float32)
    delta_ref = rows - sc.rows.astype(np.float32)
    assert np.max(np.abs(delta_dp - delta_ref)) <= 1e-6 * max(1.0, np.abs(delta_ref).max()) + 1e-9


def test_allreduce_grads_single_process_is_identity():
    from paper_2507_04004_b200 import parallel as PAR
    rows = torch.randn(10, 64)
    rows[:, 59:] = 0
    ref = rows.clone()
    touched = torch.tensor([1, 0, 1, 0, 0, 1, 0, 0, 0, 1], dtype=torch.uint8)
    PAR.allreduce_grads(rows, touched)
    assert torch.equal(rows, ref)
    assert touched.tolist() == [1, 0, 1, 0, 0, 1, 0, 0, 0, 1]
