import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B
print(B.debug_ric_step_cycles(int(sys.argv[1]) if len(sys.argv) > 1 else 512, True))
