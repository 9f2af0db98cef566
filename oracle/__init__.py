"""CPU oracle for the MQ-GNN GraphSAGE hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy, the algorithm of the reference
``mqpipe`` package (``/root/reference/pkg/src/mqpipe``) for the one path this
repository accelerates: GNS-biased node-wise sampling + relabel, feature
gather, SAGE forward/backward, summed softmax-CE, Adam/SGD and the RaCoM
window/sync arithmetic.  Every function cites the reference ``file:line`` it
follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``bench.py --impl reference``) may import it, and only as the
checker / CPU baseline.  The product package ``paper_2601_04707_b200`` never
imports this package; its compute path is the CUDA C-ABI library and fails
loudly when that library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
running the *reference itself* (imported from ``/root/reference/pkg/src``)
under the injected Philox draw contract — see ``tests/golden/make_golden.py``
and ``tests/test_oracle_golden.py`` — and the Philox generator against the
Random123 known-answer vectors.
"""
