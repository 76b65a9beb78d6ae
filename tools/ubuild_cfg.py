"""U-build / gradient device ms for a few n under the current GIVENS_RING_W (dev aid, not the bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2106_00003_b200 as g
ns = tuple(int(x) for x in sys.argv[1:]) or (1024, 2048)
print(os.environ.get("GIVENS_RING_W", "default"), bench.ubuild_table(g, torch, synth, torch.device("cuda:0"), ns=ns))
