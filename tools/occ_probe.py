"""Print the plan (kernel, slots, smem, occupancy) chosen for a config under
different shared-memory budgets (OCPQP_SMEM_KB)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2003_02547_b200 import _native as nat
    from paper_2003_02547_b200.generators import make_batch
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    b = make_batch(cfg, batch=int(sys.argv[2]) if len(sys.argv) > 2 else None)
    for kb in [None] + [int(x) for x in sys.argv[3:]]:
        if kb is None:
            os.environ.pop("OCPQP_SMEM_KB", None)
        else:
            os.environ["OCPQP_SMEM_KB"] = str(kb)
        print(kb, nat.Plan(b, b.B).info(), flush=True)


if __name__ == "__main__":
    main()
