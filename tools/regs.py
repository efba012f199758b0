"""Print registers / spills per kernel from paper_1909_07909_b200/build.log (ptxas -v)."""
import re, subprocess, sys
log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1909_07909_b200/build.log").read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur).replace("hm::", "")
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:<48} regs={m.group(1):>4} spill={spill}")
        cur = None
