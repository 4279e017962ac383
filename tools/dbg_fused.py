import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import TINY
from test_gpu_decode import SCHEDS, _setup
w, ref, plug = _setup(TINY, SCHEDS["c7f"])
tb = plug.table
print("tasks of sm3:", [(tt.TYPE_NAMES[int(t[0])], int(t[1])) for t in tb.tasks_of(3)], "begin", tb.sm_begin[3])
try:
    out = plug.decode_step(5, 0, want_logits=True); plug.check()
    want = ref.step([5],[0])[0].numpy()
    print("err", np.abs(out.logits[0].cpu().numpy()-want).max())
except Exception as e:
    print("ERR", e)
    import re
    m = re.search(r"task=(\d+)", str(e))
    if m:
        ti = int(m.group(1)); print("task", ti, list(tb.tasks[ti]))
