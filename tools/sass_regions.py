"""Static SASS instruction count of a kernel per source-line region (nvdisasm -g output).
usage: python tools/sass_regions.py file.sass kernel_substring name:a-b [name:a-b ...]"""
import re, sys, collections
path, kern = sys.argv[1], sys.argv[2]
regs = [(r.split(":")[0], *map(int, r.split(":")[1].split("-"))) for r in sys.argv[3:]]
fn = cur = None
cnt = collections.Counter()
for line in open(path):
    m = re.match(r'\s*\.text\.(\S+):', line)
    if m:
        fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if fn and kern in fn and re.match(r'\s*/\*[0-9a-f]{4,}\*/', line):
        lab = "other(" + (cur[0] if cur else "?") + ")"
        if cur and cur[0] == "fused.cu":
            for nm, a, b in regs:
                if a <= cur[1] < b:
                    lab = nm
                    break
        cnt[lab] += 1
for k, v in sorted(cnt.items(), key=lambda x: -x[1]):
    print(f"{v:6d} {k}")
