import os, sys, argparse
sys.path.insert(0, os.getcwd())
import torch
import bench
torch.cuda.set_device(0)
args = argparse.Namespace(config="C4", warmup=3, steps=3, no_cpu=True, no_sharded=True, gpus=1, impl="ours")
for rep in range(2):
    r = bench.run_ours(args, 0, 1)
    print("fast", r["fast"]["ms"], "step", r["ms_step"], "e2e", r["e2e_ms"])
