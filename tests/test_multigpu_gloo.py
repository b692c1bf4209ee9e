"""CPU, world_size 2 (gloo): the exchange plumbing of the sharded product.

The sharded kernels themselves are tested on one GPU as virtual ranks
(tests/test_gpu_parity.py::test_sharded_*); here the multi-process exchange
(torch.distributed all_to_all_single per prime, shard.torch_all_to_all) is
checked against the layout contract of shard.exchange_slices that the kernels
and LocalExchange rely on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _Info:
    def __init__(self, primes, shard_words, world):
        self.primes, self.shard_words, self.peer_words = primes, shard_words, shard_words // world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tags(rank, primes, shard_words):
    return [[(rank << 24) | (q << 20) | i for i in range(shard_words)] for q in range(primes)]


def _worker(rank, world, port, primes, shard_words, grouped, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1612_05778_b200.shard import torch_all_to_all, torch_exchange_grouped
    send = torch.tensor(_tags(rank, primes, shard_words), dtype=torch.int32)
    recv = torch.empty_like(send)
    if grouped:        # the NCCL path's grouped point-to-point exchange (two at once, as after k_low)
        send2 = send + 7
        recv2 = torch.empty_like(send)
        torch_exchange_grouped([(send, recv), (send2, recv2)], world)
        out[rank] = (recv.numpy().copy(), (recv2 - 7).numpy().copy())
    else:
        torch_all_to_all(send, recv, world)
        out[rank] = (recv.numpy().copy(),)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,primes,shard_words,grouped",
                         [(2, 3, 64, False), (2, 1, 16, False), (2, 3, 64, True), (3, 2, 48, True)])
def test_torch_exchange_matches_layout_contract(world, primes, shard_words, grouped):
    from paper_1612_05778_b200.shard import exchange_slices
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), primes, shard_words, grouped, out), nprocs=world, join=True)
    info = _Info(primes, shard_words, world)
    sends = [np.array(_tags(r, primes, shard_words), dtype=np.int32).reshape(-1) for r in range(world)]
    exp = [np.zeros(primes * shard_words, dtype=np.int32) for _ in range(world)]
    for s, t, q, so, do, w in exchange_slices(world, info):
        exp[t][do:do + w] = sends[s][so:so + w]
    for r in range(world):
        for got in out[r]:
            assert np.array_equal(got.reshape(-1), exp[r])


def _prime_worker(rank, world, port, P, shard_words, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1612_05778_b200.shard import prime_blocks, torch_prime_exchange
    blocks = prime_blocks(P, world)
    q0, nq = blocks[rank]
    S = shard_words * world
    grids = [torch.tensor([((q0 + lq) << 20) | i for i in range(S)], dtype=torch.int32) for lq in range(nq)]
    gathered = torch.full((P, shard_words), -1, dtype=torch.int32)
    torch_prime_exchange(grids, gathered, blocks, world)
    out[rank] = gathered.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P,shard_words", [(2, 3, 16), (2, 6, 8), (3, 4, 8), (2, 2, 32)])
def test_prime_exchange_matches_layout_contract(world, P, shard_words):
    # the prime split's one exchange: rank t gathers block t of every prime's
    # grid as [P][shard_words] (shard.prime_exchange_slices, tc_prime_final)
    from paper_1612_05778_b200.shard import prime_exchange_slices
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_prime_worker, args=(world, _free_port(), P, shard_words, out), nprocs=world, join=True)
    seen = {t: np.zeros((P, shard_words), dtype=bool) for t in range(world)}
    for s, t, q, lq, do, w in prime_exchange_slices(world, P, shard_words):
        exp = np.array([(q << 20) | (t * shard_words + i) for i in range(w)], dtype=np.int32)
        assert np.array_equal(out[t].reshape(-1)[do:do + w], exp)
        seen[t][q] = True
    for t in range(world):
        assert seen[t].all()
