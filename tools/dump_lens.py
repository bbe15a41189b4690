"""Write the C4 sweep's lengths (C1 law, 8 ranks, seed 1, step 0) as int64 (diagnostics)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_06001_b200 import datagen  # noqa: E402

n = int(sys.argv[1])
ids, lens = datagen.metadata("c1", 8, seed=1, step=0, per_rank=n // 8)
np.concatenate(lens).astype(np.int64).tofile(sys.argv[2])
