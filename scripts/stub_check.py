"""Runs the ctypes stub in INTEGRATION.md §2 verbatim (GPU): the documented
binding must work as written."""
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "INTEGRATION.md")).read()
i = s.index("```python", s.index("## 2. Python (ctypes) stub")) + len("```python")
os.chdir(ROOT)
ns = {}
exec(s[i:s.index("```", i)], ns)
print("stub ok: exact entries", ns["n"].value, "tvd", ns["tvd"].value)
