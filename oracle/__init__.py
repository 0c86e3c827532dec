"""TEST INFRASTRUCTURE ONLY: CPU oracle of the checking stage (see
mk_oracle.c).  Imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg."""
