"""CPU fp64 ORACLE for the recycled shifted solver of arXiv 2306.15049.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package. The product path (`paper_2306_15049_b200`) never imports it and
shares no code with it; the only module both sides use is `rsk_synth`
(seeded raw inputs, no method arithmetic).

Plain, slow, obviously-correct numpy code written from PAPER.md (cited as
P:<line>, with section / equation labels) and the readings of SURVEY.md
§8(c) listed in DESIGN.md:

  operators.py  O1  C, C^T, A = C^T C, L = [Dx; Dy], E_k = L^T W_k L,
                    A_gamma = A + gamma E_k, IRN weights, the data d, b
  dense.py      O2/O3 dense assembly and small dense tools (numpy.linalg)
  defcg.py      O4  deflated CG for one shift (the paper's recycling
                    inner solve in CG form, reading G1 / D1)
  recycle.py    O5  principal space (Alg. 1, eq:widetildeU, eq:tildeUupdate),
                    anchoring (eq:establishU), initial guesses (eq:orthupdate),
                    shift groups and local spaces (Alg. 2-4)
  pipeline.py   O6  L-curve corner, IRN outer loop (Alg. 5)

Parity pins live in tests/test_oracle_*.py (run with -m "not gpu").
Every function here is pinned there; nothing is "parity unpinned" except the
end-to-end matvec counts against the paper, whose figures were lost
 -- see DESIGN.md.
"""
