import sys; sys.path.insert(0, ".")
import torch; torch.cuda.init()
from bench import _fp32_peak
print(_fp32_peak())
