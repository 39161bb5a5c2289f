// Host-side sampling profiler for the native control plane (no perf in the
// image).  LD_PRELOAD it; SIGPROF every SAMPLER_US microseconds of CPU time
// records the interrupted PC and a short backtrace; at exit the samples and
// /proc/self/maps go to $SAMPLER_OUT.<pid>.  tools/sampler_report.py symbolises.
//   gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c
#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/syscall.h>
#include <sys/time.h>
#include <time.h>
#include <ucontext.h>
#include <unistd.h>

#define MAXS (1 << 20)
#define DEPTH 12
static uintptr_t g_s[MAXS][DEPTH];
static volatile int g_n;
static volatile int g_on;

static void on_prof(int sig, siginfo_t *si, void *uc_) {
    (void)sig;
    (void)si;
    if (!g_on) return;
    int i = __sync_fetch_and_add(&g_n, 1);
    if (i >= MAXS) return;
    ucontext_t *uc = (ucontext_t *)uc_;
    g_s[i][0] = (uintptr_t)uc->uc_mcontext.gregs[REG_RIP];
    void *bt[DEPTH + 2];
    int n = backtrace(bt, DEPTH + 2);
    // frames 0/1 are this handler and the signal trampoline
    for (int k = 1; k < DEPTH; ++k) g_s[i][k] = (k + 1 < n) ? (uintptr_t)bt[k + 1] : 0;
}

// also callable (ctypes) to (re)arm around the region of interest, in case
// a library replaced the handler after load
void sampler_start(void) {
    if (!getenv("SAMPLER_OUT")) return;
    void *warm[4];
    backtrace(warm, 4);  // load libgcc's unwinder outside the handler
    struct sigaction sa;
    memset(&sa, 0, sizeof sa);
    sa.sa_sigaction = on_prof;
    sa.sa_flags = SA_SIGINFO | SA_RESTART;
    sigaction(SIGPROF, &sa, NULL);
    int us = getenv("SAMPLER_US") ? atoi(getenv("SAMPLER_US")) : 200;
    struct itimerval it = {{0, us}, {0, us}};
    setitimer(ITIMER_PROF, &it, NULL);
    g_on = 1;
}

__attribute__((constructor)) static void start(void) { sampler_start(); }

// Wall-clock sampling of the CALLING thread only (a CLOCK_MONOTONIC hrtimer
// aimed at this thread): microsecond resolution, blocked time included.
// ITIMER_PROF fires at scheduler-tick granularity and on whichever thread
// burns CPU (e.g. a spinning worker), which blurs a ~1 us/event control plane.
void sampler_start_thread(int us) {
    if (!getenv("SAMPLER_OUT")) return;
    struct itimerval off = {{0, 0}, {0, 0}};
    setitimer(ITIMER_PROF, &off, NULL);
    struct sigevent sev;
    memset(&sev, 0, sizeof sev);
    sev.sigev_notify = SIGEV_THREAD_ID;
    sev.sigev_signo = SIGPROF;
    sev._sigev_un._tid = (pid_t)syscall(SYS_gettid);
    timer_t t;
    if (timer_create(CLOCK_MONOTONIC, &sev, &t) != 0) return;
    struct itimerspec its;
    its.it_interval.tv_sec = 0;
    its.it_interval.tv_nsec = (long)us * 1000;
    its.it_value = its.it_interval;
    timer_settime(t, 0, &its, NULL);
}

// pause (0) / resume (1) recording without disarming the timer
void sampler_enable(int on) { g_on = on; }

__attribute__((destructor)) static void stop(void) {
    const char *out = getenv("SAMPLER_OUT");
    if (!out) return;
    g_on = 0;
    struct itimerval it = {{0, 0}, {0, 0}};
    setitimer(ITIMER_PROF, &it, NULL);
    if (g_n == 0) return;  // children (compilers, helpers) inherit the env
    char path[4096];
    snprintf(path, sizeof path, "%s.%d", out, (int)getpid());
    FILE *f = fopen(path, "w");
    if (!f) return;
    int n = g_n < MAXS ? g_n : MAXS;
    fprintf(f, "samples %d\n", n);
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < DEPTH; ++k) fprintf(f, "%lx%c", (unsigned long)g_s[i][k], k + 1 < DEPTH ? ' ' : '\n');
    }
    fprintf(f, "maps\n");
    FILE *m = fopen("/proc/self/maps", "r");
    char line[4096];
    while (m && fgets(line, sizeof line, m)) fputs(line, f);
    if (m) fclose(m);
    fclose(f);
}
