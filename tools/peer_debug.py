"""Run one PeerSlab case under torchrun (dev aid)."""
import os, sys, traceback
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch
import test_peer_slab as t
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
try:
    t._worker(rank, world, int(os.environ["MASTER_PORT"]), 2, 1, (256, 1024), 5, "/tmp")
    print(f"rank {rank} ok", flush=True)
except Exception:
    traceback.print_exc()
