"""Segment timers inside NodePayload::transfer_posted (DIAGNOSTIC ONLY).

Writes an instrumented copy of csrc/host/payload.cpp to build/hostprof_seg/,
with a steady_clock stamp before each marked statement, builds it with
tools/hostprof/store_path_host.cpp + kvx_stub.cpp (no GPU) and prints the
mean microseconds per posting spent between consecutive marks.

usage: python tools/hostprof/segments.py [reps]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "build", "hostprof_seg")
MARKS = [  # (statement the stamp goes in front of, label of the segment it opens)
    ("  const Row* have = find_row(tr.session, tr.layer);", "scan source rows"),
    ("  if (f.blocks.empty()) {\n    free_flights_.push_back(slot);", "empty check"),
    ("  alloc_n(dest, f.blocks.size(), pages);", "alloc_n"),
    ("  if (dest == kHostPool || dest == kDiskPool) sort_pages(pages);", "sort (host / disk pools)"),
    ("  f.pages.resize(pages.size());", "destination refs"),
    ("  std::sort(waits.begin(), waits.end());", "waits + issue"),
    ("  kvx_check(kvx_event_create(&f.event), \"event\");", "flight event"),
    ("  {\n    Row& r = row(tr.session, tr.layer);", "row + coming marks"),
    ("  moved_[7] += f.blocks.size() * page_bytes_;", None),
]


def main():
    reps = sys.argv[1] if len(sys.argv) > 1 else "5"
    os.makedirs(OUT, exist_ok=True)
    src = open(os.path.join(ROOT, "paper_2412_16434_b200/csrc/host/payload.cpp")).read()
    i = src.index("void NodePayload::transfer_posted(")
    body = src[i:]
    for k, (stmt, _) in enumerate(MARKS):
        assert stmt in body, stmt
        body = body.replace(stmt, f"  SEG_MARK({k});\n" + stmt, 1)
    labels = ", ".join(f'"{m[1]}"' for m in MARKS[:-1])
    hdr = f"""#include <chrono>
#include <cstdio>
static double g_seg[16]; static long g_posts; static std::chrono::steady_clock::time_point g_t;
#define SEG_MARK(k) do {{ auto n_ = std::chrono::steady_clock::now(); \\
  if ((k) > 0) g_seg[(k) - 1] += std::chrono::duration<double, std::micro>(n_ - g_t).count(); \\
  else ++g_posts; g_t = n_; }} while (0)
extern "C" void seg_dump() {{ static const char* l[] = {{{labels}}};
  for (int k = 0; k < {len(MARKS) - 1}; ++k) std::printf("  %-26s %7.2f us per posting\\n", l[k], g_seg[k] / (g_posts ? g_posts : 1)); }}
"""
    open(os.path.join(OUT, "payload.cpp"), "w").write(hdr + src[:i] + body)
    main_src = open(os.path.join(ROOT, "tools/hostprof/store_path_host.cpp")).read()
    main_src = main_src.replace("int main(int argc, char** argv) {", 'extern "C" void seg_dump();\nint main(int argc, char** argv) {')
    main_src = main_src.replace("  return 0;\n}", "  seg_dump();\n  return 0;\n}")
    open(os.path.join(OUT, "main.cpp"), "w").write(main_src)
    exe = os.path.join(OUT, "store_path_seg")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(OUT, "main.cpp"), f"{ROOT}/tools/hostprof/kvx_stub.cpp", os.path.join(OUT, "payload.cpp"),
                    f"{ROOT}/paper_2412_16434_b200/csrc/host/kvstore.cpp",
                    f"{ROOT}/paper_2412_16434_b200/csrc/host/costmodel.cpp", "-o", exe], check=True)
    subprocess.run([exe, reps], check=True)


if __name__ == "__main__":
    main()
