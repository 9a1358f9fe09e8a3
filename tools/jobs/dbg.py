import sys; sys.path.insert(0,'.')
import torch
from paper_1905_01141_b200 import crn
torch.zeros(1).cuda()
print(crn.decode_kernel_info())
print(crn.workspace_bytes(), crn.lib().crn_last_error())
