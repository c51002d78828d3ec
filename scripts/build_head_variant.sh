# Build the committed HEAD (or $1) into paper_1805_06572_b200/lib/var_head.so for A/B runs
set -e
REV=${1:-HEAD}
rm -rf /tmp/ffca_wt && git -C /root/repo worktree prune && git -C /root/repo worktree add -f /tmp/ffca_wt $REV > /dev/null
(cd /tmp/ffca_wt && python -m paper_1805_06572_b200.build > /tmp/ffca_wt_build.log 2>&1)
cp /tmp/ffca_wt/paper_1805_06572_b200/lib/libfastfca_b200.so /root/repo/paper_1805_06572_b200/lib/var_head.so
git -C /root/repo worktree remove --force /tmp/ffca_wt
echo built var_head.so from $REV
