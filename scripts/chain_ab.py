"""A/B of the persistent decode-layer chain kernel vs one kernel per projection.

    python scripts/chain_ab.py out.pt [layers] [R]     (run under PL_CHAIN=0 and =1)

Greedy prefill + decode steps of a truncated Llama-3-8B-shape stage (packed weights);
saves the ids and the final-normed rows so two runs can be compared.
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402
from paper_2507_05043_b200.spec import prompt_tokens  # noqa: E402

out = sys.argv[1]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
R = int(sys.argv[3]) if len(sys.argv) > 3 else 8
spec = LLAMA3_8B.with_(num_layers=L)
lens = [40 + 7 * r for r in range(R)]
steps = 5
exe = StageExecutor(spec, 0, (0, L), True, True, torch.device("cuda", 0), seed=0, max_tokens=sum(lens),
                    max_reqs=R, max_ctx=max(lens) + steps, num_blocks=sum(-(-(n + steps) // 64) for n in lens),
                    n_slots=1)
ids, hn = exe.greedy([prompt_tokens(0, r, n, spec.vocab) for r, n in enumerate(lens)], steps)
torch.save({"ids": torch.from_numpy(ids), "hn": hn}, out)
print("ids", ids[:, :].tolist()[:3])
