"""Global loads scheduled before griddepcontrol.wait (ACQBULK) in the SASS of
the PDL-launched kernels of libfcg.so.

ptxas treats ld.global.nc (LDG.CONSTANT: __ldg and const __restrict__
pointers) as invariant and may hoist it above griddepcontrol.wait, which
then reads the predecessor kernel's output before that kernel has finished.
A load of step data must never precede ACQBULK.

    python tools/check_pdl.py [libfcg.so]      (exit 1 if any)
"""
import re
import subprocess
import sys

PDL_KERNELS = ("k_edge_geom", "k_edge_fwd_tc", "k_edge_bwd_tc", "k_edge_bwd64", "k_edge_fwd64",
               "k_edge_bwd_fm", "k_edge_bwd_fmws", "k_edge_fwd_ws", "k_node_linear_tc",
               "k_node_post_tc", "k_node_post_bwd_tc", "k_readout_tc", "k_node_post_pre_tc",
               "k_node_post_readout_tc", "k_node_prebwd_postbwd_tc",
               "k_noise_baoa_ring", "k_prior",
               "k_embed", "k_forces_finish", "k_scan_rows", "k_nbr_assemble",
               "k_fill_masks", "k_rev_masks")


def early_loads(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    res, fn, seen_wait = {}, None, False
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1) if any(k in m.group(1) for k in PDL_KERNELS) else None
            seen_wait = False
            if fn:
                res[fn] = {"wait": False, "early": [], "nc": 0}
            continue
        if not fn:
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if not m:
            continue
        ins = m.group(2)
        if "ACQBULK" in ins:
            seen_wait = True
            res[fn]["wait"] = True
        elif not seen_wait and re.search(r"\bLDG\b|\bLDG\.|\bLD\.E", ins):
            res[fn]["early"].append(f"{m.group(1)} {ins.strip()}")
        if re.search(r"\bLDG\.\S*CONSTANT", ins):
            res[fn]["nc"] += 1
    return res


def main(lib):
    res = early_loads(lib)
    bad = 0
    for fn, r in sorted(res.items()):
        # nc loads after the wait are reported, not failed (constant tables
        # such as sincosf's reduction table are legitimately read-only)
        status = "ok" if r["wait"] and not r["early"] else "BAD"
        bad += status == "BAD"
        print(f"{status:3s} {fn[:70]:70s} wait={r['wait']} early_loads={len(r['early'])} nc_loads={r['nc']}")
        for x in r["early"][:6]:
            print("      ", x)
    return 1 if bad or not res else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1] if len(sys.argv) > 1 else "paper_2602_13140_b200/libfcg.so"))
