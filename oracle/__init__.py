"""CPU ORACLE — test infrastructure only, never a product path.

This package restates, on the CPU, the reference's algorithm for the Round
Attention hot path (`/root/reference/pkg/src/roundkv/...`, cited file:line in
every function).  It exists to CHECK the CUDA path:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
  `--impl reference` legs may import it;
* the product package (`paper_2502_15294_b200`) never imports it and has no
  CPU fallback — it fails loudly when `librk.so` is missing.

Parity pinning: the restatement is checked bit-for-bit / within 1e-12 against
golden vectors produced by the real reference imported in the build container
(`tools/make_golden.py` -> `tests/golden/*.npz`, see `tests/test_oracle_golden.py`).

Modules
  attention  -- `attention_forward` kernel contract (fp64), GQA expansion
  rounds     -- Eq. 1 aggregation, normalize, selection strategies, numpy-exact
                pairwise sums, tiered-store ledger, Eq. 2 memory model
  model      -- the reference's toy attention model and `RoundPipeline.run_turn`
  cref       -- ctypes binding of `attn_ref.c` (threaded C restatement of the
                Cython kernel) used as the CPU baseline port
  refkernel  -- loader for the reference's own Cython kernel compiled from
                /root/reference into `oracle/_ref/` (CPU baseline "reference")
"""
