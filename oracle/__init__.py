"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TANQ-Sim hot path.

A plain, slow, obviously-correct dense density-matrix simulator written from
the paper (arXiv 2404.13184, /root/reference/PAPER.md, cited as P:<line>).  It
computes Eq. (dmsim) rho_out = G_{m-1} ... (G_0 rho_in G_0^dag) ... G_{m-1}^dag
 with every noisy gate applied as its sequence of Kraus channels
xi(rho) = sum_i K_i rho K_i^dag, acting on the dense 2^n x 2^n matrix
rho[r][c] (row-major, NOT vec, no superoperators, no fusion, no layout tricks).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2404_13184_b200``) never imports it and shares no code,
headers or tables with it.

Modules
  channels.py    gate unitaries, Kraus channels, noise binding (numpy)      -- pinned
  dense.c        block-wise Kraus / depolarizing application, probabilities,
                 Pauli expectation, readout (C + OpenMP)                   -- pinned
  dense.py       ctypes driver for dense.c; run(circuit, noise) -> rho      -- pinned
  kron_small.py  independent n<=5 full-Kronecker cross-check (numpy)        -- pinned
  statevector.py brute-force state vector for noiseless pins (numpy)        -- pinned

"parity unpinned": the noise-model *conventions* (readings R4-R6,
R10, R11) are fixed by our reading, not by the paper; each channel in
isolation is pinned to its closed form, their composition order is not.
"""
