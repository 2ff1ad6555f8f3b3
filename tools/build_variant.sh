# Build a variant of the library with extra nvcc flags into exp/<name>/ (A/B runs:
# LBM_PKG_ROOT=exp/<name> python tools/sweep_bench.py ...).  usage: build_variant.sh <name> <flags...>
name=$1; shift
d=exp/$name/paper_2208_05429_b200; mkdir -p $d
cp paper_2208_05429_b200/__init__.py paper_2208_05429_b200/build.py $d/
NVCC_EXTRA="$*" python - <<'PY' "$d"
import os, subprocess, sys
sys.path.insert(0, "paper_2208_05429_b200")
import build as b
out = os.path.join(sys.argv[1], "liblbm_b200.so")
cmd = [b.NVCC, *b.FLAGS, *os.environ["NVCC_EXTRA"].split(), "-I", "include", *b.sources(), "-o", out, "-ldl"]
subprocess.check_call(cmd, stderr=subprocess.DEVNULL)
print(out)
PY
