"""CPU oracle for the policy-selected AllReduce hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything here.  The product path
(``paper_2603_11438_b200``, ``libpolar.so``) never imports, links or executes it,
and this package never imports the product path: the two share no code, tables
or constants.

Modules
-------
``allreduce``  rank-ordered sum/max/min reduction (SURVEY.md §8(c) "Definition
               of the result"; PAPER.md L106-107 AllReduce as a primitive).
``policy``     the policy table's size -> (algorithm, protocol, channels) mapping
               as a plain linear scan (
               SPEC.md L336-345), with its own transcription of the library's
               built-in default table.
``metrics``    algBW / busBW arithmetic.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
(brute force, closed forms, the paper's worked examples).  Nothing is "parity
unpinned".
"""
