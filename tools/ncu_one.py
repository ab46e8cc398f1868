"""One un-graphed streaming call (one launch per op) for ncu captures of a single layer:
  ncu --set full -k regex:conv_tc_kernel --launch-skip K --launch-count 1 \\
      python tools/ncu_one.py CFG [STREAMS] [fp32|bf16]
K = the layer's index among the call's tensor-core launches (see Plan.launch_names)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_07064_b200 import configs  # noqa: E402
from paper_2204_07064_b200.runtime import Plan, StreamState  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
S = int(sys.argv[2]) if len(sys.argv) > 2 else configs.CONFIGS[cfg]["streams"]
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
m = configs.build(cfg)
plan = Plan(m, precision=prec)
F = configs.CONFIGS[cfg]["frames"]
st = StreamState(plan, S, F)
st.set_graphs(False)
num, den, cout = plan.sink
x = torch.randn(S, m.in_channels, F, device="cuda")
y = torch.empty(S, cout, F * num // den, device="cuda")
if os.environ.get("NCU_ONE_LIST"):
    print("\n".join(n for n in st.launch_names(F)))
st.process_buffer(x, y, F)
torch.cuda.synchronize()
print("ok")
