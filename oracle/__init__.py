"""TEST INFRASTRUCTURE: CPU checkers (C restatement + compiled reference).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package; the product path (paper_2505_10168_b200) never does.
"""
