"""One-off refactor helper: turn `__global__ K(params) {body}` into a force-inlined
`K_body` (big structs by const reference) plus a thin kernel calling it."""
import re, sys

REF = {"GridView", "RotCache", "MapView"}


def split_params(p):
    out, depth, cur = [], 0, ""
    for ch in p:
        if ch in "(<[":
            depth += 1
        elif ch in ")>]":
            depth -= 1
        if ch == "," and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip():
        out.append(cur.strip())
    return out


def bodyize(src, name):
    m = re.search(r"(template <[^>]*>\n)?__global__ void (__launch_bounds__\([^)]*\) )?" + name + r"\(", src)
    assert m, name
    start = m.start()
    tmpl = m.group(1) or ""
    lb = m.group(2) or ""
    i = m.end()
    depth = 1
    while depth:
        if src[i] == "(":
            depth += 1
        elif src[i] == ")":
            depth -= 1
        i += 1
    params = src[m.end():i - 1]
    assert src[i:i + 2] == " {", (name, src[i:i + 10])
    j = i + 2
    depth = 1
    while depth:
        if src[j] == "{":
            depth += 1
        elif src[j] == "}":
            depth -= 1
        j += 1
    body = src[i + 2:j - 1]
    plist = split_params(params)
    bparams, names = [], []
    for p in plist:
        toks = p.replace("*", " * ").replace("&", " & ").split()
        nm = toks[-1]
        names.append(nm)
        ty = toks[0] if toks[0] != "const" else toks[1]
        if ty in REF and "*" not in p and "&" not in p:
            bparams.append(f"const {ty}& {nm}")
        else:
            bparams.append(p)
    targs = ""
    if tmpl:
        targs = "<" + ", ".join(t.split()[-1] for t in tmpl[len("template <"):-2].split(",")) + ">"
    ind = " " * len(f"__device__ __forceinline__ void {name}_body(")
    new = (f"{tmpl}__device__ __forceinline__ void {name}_body(" + (",\n" + ind).join(bparams) + ") {" + body + "}\n\n"
           f"{tmpl}__global__ void {lb}{name}({params}) {{\n  {name}_body{targs}({', '.join(names)});\n}}")
    return src[:start] + new + src[j:]


if __name__ == "__main__":
    path = sys.argv[1]
    s = open(path).read()
    for k in sys.argv[2:]:
        s = bodyize(s, k)
    open(path, "w").write(s)
