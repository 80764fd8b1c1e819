"""fp64 CPU oracle for WallFacer multi-ring attention (arXiv 2407.00611).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2407_00611_b200``) never imports it, and
this package never imports the product path: the two share no code, only the
seeded generators in ``wf_inputs``.

Modules
-------
dense     -- Eq. 1 softmax attention forward and its exact gradients (fp64).
blocks    -- the per-block primitives the paper's loop is built from:
             forward_iteration (online-softmax merge, Alg. 1 l.9) and the
             flash-attention backward step (§3.2.1 "Backward Propagation").
topology  -- Alg. 2 get_init_send, its inverse, Alg. 3 get_P2P_config.
sharding  -- §3.5 naive / zigzag dataloader.
proj      -- the QKV projection of Alg. 1 l.1 (AllGather_QKVmatmul).
schedule  -- literal simulation of Alg. 1 + the two-loop backward, rank by
             rank, with fp64 payloads and a CommTrace.

Parity pins: see DESIGN.md "Oracle pins".  Every function is pinned except
where its docstring says "parity unpinned".
"""
