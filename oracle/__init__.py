"""CPU restatement of the reference path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the CPU
baseline.  The product (paper_2010_14501_b200) never imports it and has no CPU
fallback.

* ledger.py       — the reference simulator's byte ledger (schedule.py:320-465)
                    restated independently; pinned against golden ledgers the
                    reference itself produced (tests/golden/).
* bitmask.py      — numpy packer for the ReLU sign bitmask layout.
* cpu_executor.py — torch-CPU fp32 replay of a Schedule on a traced Network:
                    forward in node order, per-stage drops/recomputes with saved
                    BN statistics, per-variant backward semantics (PAPER.md
                    App. D, 957-990), SGD.  Its numerics are pinned against
                    plain torch autograd of the same torchvision model (the
                    reference package itself has no numeric implementation:
                    "parity unpinned" by the reference).
"""
