"""C5 alternative reading (1 market x 1024 books, 100 steps) and C5 itself: device ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16508_b200 import finance as F  # noqa: E402

one = F.FinanceConfig(books=1024)
F.run_batch(one, 7, 1, 100)
print("one market ms", [round(F.run_batch(one, 7, 1, 100)[1], 3) for _ in range(3)])
F.run_batch(F.FinanceConfig(), 7, 1024, 100)
print("C5 ms", [round(F.run_batch(F.FinanceConfig(), 7, 1024, 100)[1], 3) for _ in range(3)])
