"""Run the README's Python quick start (keeps the documented API honest)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
src = open(os.path.join(ROOT, "README.md")).read().split("```python")[1].split("```")[0]
ns = {}
exec(compile(src, "README.md", "exec"), ns)
print("quickstart ok:", ns["rep"], ns["y"].shape, ns["xi"].shape, ns["f"])
