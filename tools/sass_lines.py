"""Static SASS instruction counts per source line for one kernel of a cubin (nvdisasm -g).
Usage: python tools/sass_lines.py file.cubin kernel_substring [top]"""
import collections
import re
import subprocess
import sys

cubin, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cnt = collections.Counter()
cur_fn, cur_line, infn = None, None, False
for ln in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        infn = kname in cur_fn
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if infn and re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        cnt[cur_line] += 1
print("total", sum(cnt.values()))
for (f, l), c in cnt.most_common(top):
    print(c, f, l)
