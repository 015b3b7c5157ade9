// Measurement knobs (internal.hpp Knobs).  The product library returns the defaults and never
// reads the environment; the variants build (-DACCSPMM_VARIANTS) re-reads ACCSPMM_* on every
// call so an A/B sweep can flip them between executes of one plan (tools/sweep.py).
#include <cstdlib>

#include "../internal.hpp"

namespace accspmm {

#ifdef ACCSPMM_VARIANTS
static int64_t env_i64(const char *name, int64_t dflt)
{
    const char *s = std::getenv(name);
    return s ? std::atoll(s) : dflt;
}

const Knobs &knobs()
{
    static thread_local Knobs k;
    const Knobs d;
    k.kcfg = (int)env_i64("ACCSPMM_KCFG", d.kcfg);
    k.fw = (int)env_i64("ACCSPMM_FW", d.fw);
    k.slice_major = (int)env_i64("ACCSPMM_SLICE_MAJOR", d.slice_major);
    k.l2promo = (int)env_i64("ACCSPMM_L2PROMO", d.l2promo);
    k.round_b = (int)env_i64("ACCSPMM_ROUND_B", d.round_b);
    k.l2_persist_mib = env_i64("ACCSPMM_L2_PERSIST", d.l2_persist_mib);
    k.group_cap = (int)env_i64("ACCSPMM_GROUP_CAP", d.group_cap);
    k.reorder_L = (int)env_i64("ACCSPMM_REORDER_L", d.reorder_L);
    k.reorder_H = (int)env_i64("ACCSPMM_REORDER_H", d.reorder_H);
    k.b3 = (int)env_i64("ACCSPMM_B3", d.b3);
    k.hot_bytes = env_i64("ACCSPMM_HOT_MB", d.hot_bytes >> 20) << 20;
    k.hot_l2_bytes = env_i64("ACCSPMM_HOT_L2_MB", d.hot_l2_bytes >> 20) << 20;
    return k;
}
#else
const Knobs &knobs()
{
    static const Knobs k;
    return k;
}
#endif

}  // namespace accspmm
