import sys
sys.path.insert(0, ".")
from paper_2504_09983_b200 import dc  # noqa: E402
print("pair slots", dc.lib.dc_gemm_pair_slots())
