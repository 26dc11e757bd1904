"""The NCCL communicator inside libsom (som_comm_unique_id /
som_comm_init_nccl) on one GPU (world = 1; NCCL refuses two
ranks on one device, so world > 1 runs only on a multi-GPU box):
  * SOM_XCHG_NCCL training (one step kernel + one ncclAllReduce(u64, min)
    per step, graph-replayed) reproduces the oracle, with and without the
    CUDA graphs and across a resume;
  * a document-sharded handle's errors (fp64 sum + int64 counts all-reduced)
    equal the unsharded call, and an empty shard joins the reduction."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


@pytest.mark.parametrize("graph", [True, False])
def test_nccl_exchange_training_matches_oracle(som, monkeypatch, graph):
    if not graph:
        monkeypatch.setenv("SOM_NCCL_GRAPH", "0")
    C = bank_corpus(200, 500, seed=1)
    X = C.dense()
    W0 = init_rows(X, 100, 1)
    T = 5 * 200
    with som.SOM(10, 10, 500, 0) as m:
        som.som_comm_init_nccl(m.h, 0, 1, som.som_comm_unique_id(), som.SOM_SHARD_NEURONS)
        som.som_set_exchange(m.h, som.SOM_XCHG_NCCL)
        m.set_weights(W0)
        log = np.empty(T, np.int32)
        m.train_online(X, epochs=5, alpha0=0.1, sigma0=5.0, seed=1, t_end=613, bmu_log=log[:613])
        m.train_online(X, epochs=5, alpha0=0.1, sigma0=5.0, seed=1, t_begin=613, bmu_log=log[613:])
        assert som.som_last_train_config(m.h)[1] == 8
        ms, steps, launches = som.som_last_stats(m.h)
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, 10, 10, 0, X, 5, 0.1, 5.0, 1)
    assert np.array_equal(log, logo)
    assert np.abs(W - Wo).max() <= 1e-4
    print(f" [NCCL exchange, graph={graph}: {1000 * ms / steps:.2f} us/step over {steps} steps]", end="")


def test_doc_sharded_errors_reduce(som):
    C = bank_corpus(1500, 800, seed=3)
    X = C.dense()
    W = init_rows(X, 64, 3)
    with som.SOM(8, 8, 800, 1) as m:
        m.set_weights(W)
        qe1, te1 = m.errors(X)
        q_csr1, t_csr1 = m.errors_csr(C.indptr, C.indices, C.data, C.n)
    with som.SOM(8, 8, 800, 1) as m:
        som.som_comm_init_nccl(m.h, 0, 1, som.som_comm_unique_id(), som.SOM_SHARD_DOCS)
        m.set_weights(W)
        qe, te = m.errors(X)
        assert abs(qe - qe1) <= 1e-12 * qe1 and te == te1
        q2, t2 = m.errors_csr(C.indptr, C.indices, C.data, C.n)
        assert abs(q2 - q_csr1) <= 1e-12 * q_csr1 and t2 == t_csr1
        with pytest.raises(som.SomError) as e:      # empty shard, and nobody else has rows
            som.som_errors(m.h, X, 0)
        assert e.value.status == som.SOM_EEMPTY
