"""Report the innermost FFMA loops of a kernel in a cuobjdump -sass listing.

    python tools/sass_loops.py listing.sass screen_kernelILi8
"""
import re
import sys


def main(path, needle, min_ffma=8):
    txt = open(path).read()
    for part in re.split(r"\n\s+Function : ", txt):
        head = part.split("\n", 1)[0]
        if needle not in head:
            continue
        lines = [l for l in part.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,5}\*/", l)]

        def addr(l):
            return int(re.search(r"/\*([0-9a-f]{4,5})\*/", l).group(1), 16)

        for l in lines:
            m = re.search(r"BRA (0x[0-9a-f]+)", l)
            if m and int(m.group(1), 16) < addr(l):
                tgt = int(m.group(1), 16)
                body = [x for x in lines if tgt <= addr(x) <= addr(l)]
                nf = sum("FFMA" in x for x in body)
                if nf >= min_ffma:
                    cnt = lambda s: sum(s in x for x in body)  # noqa: E731
                    print(f"{head[:60]} loop {hex(tgt)}-{hex(addr(l))} len {len(body)} "
                          f"FFMA {nf} LDG {cnt('LDG')} LDC {cnt('LDC')} SHFL {cnt('SHFL')} "
                          f"LDS {cnt('LDS')} local {cnt('STL') + cnt('LDL')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 8)
