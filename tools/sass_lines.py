"""Static SASS instruction mix of one kernel by source line (nvdisasm --print-line-info output).
usage: python tools/sass_lines.py <disasm.txt> <mangled-name-substring> [top]"""
import collections, re, sys

path, name = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None
inside = False
cnt, tot = collections.Counter(), collections.Counter()
ops = collections.defaultdict(collections.Counter)
for line in open(path):
    if line.startswith("//--") and ".text." in line:
        inside = name in line
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)".*line (\d+)', line)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        continue
    m2 = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m2 and cur:
        op = m2.group(1).split(".")[0]
        cnt[cur] += 1
        ops[cur][op] += 1
        tot[op] += 1
print(sum(tot.values()), tot.most_common(20))
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    print(v, k, dict(ops[k].most_common(5)))
