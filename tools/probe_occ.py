"""Occupancy (CTAs/SM) the runtime reports for the streaming kernels at the config ks."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1708_02845_b200 import _native as nat
lib = nat.load()
print(torch.cuda.get_device_name())
