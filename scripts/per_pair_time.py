"""Time the per-pair drop-in path (bench.per_pair_leg) alone: python scripts/per_pair_time.py [envs]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200.scenes import m16_workload

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    w = m16_workload(n + 1)
    for _ in range(2):
        print(json.dumps(bench.per_pair_leg(P, w, n)), flush=True)


if __name__ == "__main__":
    main()
