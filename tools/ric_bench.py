import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 512
print("team riccati step, cycles:", B.debug_ric_step_cycles(steps, 1))
tot, st = B.debug_ric_step_cycles(steps, 2)
print("stamped: total %.0f; S1 %.0f  S2 %.0f  S3(ldlt,K) %.0f  S4 %.0f  store+ballot %.0f" % (tot, *st))
tot, st = B.debug_ric_step_cycles(steps, 3)
print("32-lane team: total %.0f; S1 %.0f  S2 %.0f  S3(ldlt,K) %.0f  S4 %.0f  store+ballot %.0f" % (tot, *st))
