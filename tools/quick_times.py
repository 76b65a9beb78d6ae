"""Quick device timings of the headline pieces (C3 apply/backward, unitary n=1024) -- a dev aid, not the bench."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2106_00003_b200 as g
dev = torch.device("cuda:0")
print("unitary", bench.unitary_line(g, torch, synth, dev, 74.45))
