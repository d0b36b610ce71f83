"""Print the SASS of one kernel from libaidw.so (substring match on the mangled name),
or with --count, the LDL/STL lines and their position within the listing.
usage: python tools/sass_fn.py SUBSTR [--spills]"""
import re
import subprocess
import sys

so = "paper_1511_02186_b200/libaidw.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
sub = sys.argv[1]
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if sub in name:
        lines = [l for l in f.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
        print("==", name, len(lines), "instructions")
        if "--spills" in sys.argv:
            for i, l in enumerate(lines):
                if re.search(r"\b(LDL|STL)\b", l) or re.search(r"\bBRA\b", l):
                    print(i, l.split(";")[0].strip())
        else:
            print("\n".join(lines))
        break
