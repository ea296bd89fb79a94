"""The bench roofline probe launch (64 polys x 11 limbs forward Bluestein at C2), for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

ctx = bc.Context(bc.load_params("c2"))
print(bc.profile_ntt(ctx))
