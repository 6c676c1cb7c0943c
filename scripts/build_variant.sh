# Build a libadsb variant into ab/libadsb_<name>.so with extra nvcc flags (A/B runs via ADSB_LIB_PATH).
# usage: bash scripts/build_variant.sh <name> "<-Dflags>"
set -e
NAME=$1; FLAGS=$2; ROOT=$(cd "$(dirname "$0")/.." && pwd)
D=$(mktemp -d /tmp/adsb_variant_XXXX)
cp -r "$ROOT/paper_1903_09422_b200" "$ROOT/include" "$ROOT/tools" "$D/"
rm -f "$D/paper_1903_09422_b200/libadsb.so"
(cd "$D" && ADSB_NVCC_EXTRA="$FLAGS" python -m paper_1903_09422_b200.build --force > build.log 2>&1) || { cat "$D/build.log"; exit 1; }
mkdir -p "$ROOT/ab"
cp "$D/paper_1903_09422_b200/libadsb.so" "$ROOT/ab/libadsb_$NAME.so"
rm -rf "$D"
echo "built ab/libadsb_$NAME.so ($FLAGS)"
