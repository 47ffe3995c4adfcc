"""CPU oracle (test infrastructure).  See flashcg_oracle.py's header: only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use it."""
