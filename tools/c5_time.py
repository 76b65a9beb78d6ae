"""C5 shard line and n=2048 U-build gradient, device ms (dev aid, not the bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2106_00003_b200 as g
dev = torch.device("cuda:0")
r = bench.c5_shard_line(g, torch, synth, dev)
print("c5", r["fwd_ms"], r["bwd_ms"], bench.ubuild_table(g, torch, synth, dev, ns=(1120, 2048)))
