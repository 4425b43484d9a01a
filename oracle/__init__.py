"""CPU oracles — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import anything from here, and only as the checker (or as the timed
CPU baseline). The worker's product path never routes through this package.
"""
